#!/bin/bash
# GMM renormalisation with a hoisted reciprocal: GPU parity + bench A/B against tuning/lib_base.so.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
export RGBDSEG_B200_AUTOBUILD=0
timeout 900 python -m pytest tests/test_gmm_f32.py tests/test_gpu_parity.py -m gpu -q -x -k "gmm or f32 or golden or divide or kat" > gpurun_out/pytest_renorm.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_renorm.log
for st in f64 f32; do for rep in 1 2; do
for lib in "" tuning/lib_base.so; do
  tag=${lib:-new}; tag=$(basename "$tag" .so)
  RGBDSEG_B200_LIB=${lib:+$PWD/$lib} timeout 300 python bench.py --steps 60 --warmup 10 --no-e2e --no-cpu-baseline --gmm-state $st > gpurun_out/r_${st}_${tag}_$rep.json 2>/dev/null
  echo "$st $tag $rep $(python -c "import json;d=json.load(open('gpurun_out/r_${st}_${tag}_$rep.json'));print({k:(round(v['ms_per_step'],4),round(v['roofline_frac'],3)) for k,v in d['per_algo'].items()})" 2>&1)"
done; done; done

#!/bin/bash
# Benchmark tuning variants of the native library (tuning/lib_*.so) on the GPU box.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
shopt -s nullglob
for lib in "" tuning/lib_*.so; do
  tag=${lib:-default}; tag=$(basename "$tag" .so)
  RGBDSEG_B200_LIB=${lib:+$PWD/$lib} timeout 300 python bench.py --steps 60 --warmup 10 --no-e2e --no-cpu-baseline ${VARIANT_BENCH_ARGS} > gpurun_out/var_$tag.json 2> gpurun_out/var_$tag.err
  echo "$tag $(python -c "import json;d=json.load(open('gpurun_out/var_$tag.json'));print({k:(round(v['ms_per_step'],4),round(v['roofline_frac'],3)) for k,v in d['per_algo'].items()})" 2>&1)"
done

#!/bin/bash
# Tuning variants (tuning/lib_*.so) x workloads: ms/step of each bench config.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
shopt -s nullglob
for wl in ${WORKLOADS:-config1 config2 config4}; do
  for lib in "" tuning/lib_*.so; do
    tag=${lib:-default}; tag=$(basename "$tag" .so)
    RGBDSEG_B200_LIB=${lib:+$PWD/$lib} timeout 300 python bench.py --workload $wl --steps ${STEPS:-100} --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/vc_${wl}_$tag.json 2> gpurun_out/vc_${wl}_$tag.err
    echo "$wl $tag $(python -c "import json;d=json.load(open('gpurun_out/vc_${wl}_$tag.json'));print(round(d['ms_per_step'],4), {k:round(v['ms_per_step'],4) for k,v in d.get('per_algo',{}).items()})" 2>&1 | tail -1)"
  done
done

#!/bin/bash
# Opt-in f32 GMM storage: K1 occupancy variants (tuning/lib_f*.so), config 4.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export RGBDSEG_B200_AUTOBUILD=0
for lib in "" tuning/lib_f*.so; do
  tag=${lib:-default}; tag=$(basename "$tag" .so)
  RGBDSEG_B200_LIB=${lib:+$PWD/$lib} timeout 300 python bench.py --gmm-state f32 --steps 50 --warmup 5 --no-e2e \
    --no-cpu-baseline --no-verify > gpurun_out/f32.json 2>/dev/null
  echo "$tag $(python -c "import json;d=json.load(open('gpurun_out/f32.json'));p=d['per_algo']['gmm'];print(round(p['ms_per_step'],4),'ms', round(p['roofline_frac'],3), round(d['ms_per_step'],4))")"
done

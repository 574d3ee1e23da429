#!/bin/bash
# Config 1 (GMM 3/3, 640x480, cold L2): K1 occupancy variants.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export RGBDSEG_B200_AUTOBUILD=0
for lib in "" tuning/lib_gs*.so; do
  tag=${lib:-default}; tag=$(basename "$tag" .so)
  RGBDSEG_B200_LIB=${lib:+$PWD/$lib} timeout 300 python bench.py --workload config1 --steps 100 --warmup 5 --no-e2e \
    --no-cpu-baseline --no-verify > gpurun_out/g1.json 2>/dev/null
  echo "$tag $(python -c "import json;d=json.load(open('gpurun_out/g1.json'));p=d['per_algo']['gmm'];print(round(p['ms_per_step']*1e3,2),'us', round(p['roofline_frac'],3))")"
done

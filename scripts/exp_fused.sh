#!/bin/bash
# Fused small-frame PBAS variants (tuning/lib_*.so), configs 2-3 at T = t_lower.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export RGBDSEG_B200_AUTOBUILD=0
for lib in "" tuning/lib_*.so; do
  tag=${lib:-default}; tag=$(basename "$tag" .so)
  for wl in config2 config3; do
    RGBDSEG_B200_LIB=${lib:+$PWD/$lib} timeout 300 python bench.py --workload $wl --steps 50 --warmup 5 --no-e2e \
      --no-cpu-baseline --no-verify > gpurun_out/small.json 2>/dev/null
    echo "$tag $wl $(python -c "import json;d=json.load(open('gpurun_out/small.json'));p=d['per_algo']['pbas'];y=d.get('pbas_young') or {};print(round(p['ms_per_step']*1e3,1),'us', round(p['roofline_frac'],3), 'young', round(y.get('ms_per_step',0)*1e3,1), round(y.get('roofline_frac',0),3))")"
  done
done

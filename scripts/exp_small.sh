#!/bin/bash
# Small-frame PBAS (configs 2 and 3, one stream, steady state T = t_lower):
# K2 variants and strip heights.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export RGBDSEG_B200_AUTOBUILD=0
for wl in config2 config3; do
  for v in "rows" "strips" "unfused" "fused" "auto"; do
    mode=${v%%:*}; sh=${v#*:}; [ "$sh" = "$v" ] && sh=""
    RGBDSEG_STRIP_H=$sh timeout 300 python bench.py --workload $wl --steps 50 --warmup 5 --no-e2e \
      --no-cpu-baseline --no-verify --k2-mode $mode > gpurun_out/small.json 2>/dev/null
    echo "$wl $v $(python -c "import json;d=json.load(open('gpurun_out/small.json'));p=d['per_algo']['pbas'];print(round(p['ms_per_step']*1e3,1),'us', round(p['roofline_frac'],3), d['model_age']['pbas_k2_variant'])")"
  done
done

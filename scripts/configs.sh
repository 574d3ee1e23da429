#!/bin/bash
# Bench lines for every BASELINE config that fits one GPU (configs 1-5).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for wl in config1 config2 config3 config4 config5; do
  timeout 600 python bench.py --workload $wl --steps ${STEPS:-200} --warmup 10 --no-cpu-baseline ${CONFIG_ARGS} \
    > gpurun_out/cfg_$wl.json 2> gpurun_out/cfg_$wl.err
  echo "$wl $(python -c "import json;d=json.load(open('gpurun_out/cfg_$wl.json'));print(round(d['value'],1), round(d['ms_per_step'],4), {k:(round(v['ms_per_step'],4),round(v.get('roofline_frac') or 0,3)) for k,v in d.get('per_algo',{}).items()}, d.get('e2e') and round(d['e2e']['value'],1))" 2>&1 | tail -1)"
done

#!/bin/bash
# GMM / PBAS co-scheduling sweep: occupancy caps via dynamic shared memory
# (RGBDSEG_GMM_SMEM / RGBDSEG_PBAS_SMEM bytes per block) and stream priority.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
run() {  # tag gmm_smem pbas_smem prio
  RGBDSEG_GMM_SMEM=$2 RGBDSEG_PBAS_SMEM=$3 timeout 300 python bench.py --steps 60 --warmup 10 --no-e2e \
    --no-cpu-baseline --stream-priority $4 > gpurun_out/co_$1.json 2> gpurun_out/co_$1.err
  echo "$1 gmm_smem=$2 pbas_smem=$3 prio=$4 $(python -c "import json;d=json.load(open('gpurun_out/co_$1.json'));print(round(d['ms_per_step'],4), round(d['value'],1))" 2>&1 | tail -1)"
}
run base 0 0 0
run g3 60000 0 0
run g2 100000 0 0
run g2p 100000 0 1
run g1 200000 0 0
run p2 0 100000 0
run g3p1 60000 200000 0
run g2p2 100000 100000 0

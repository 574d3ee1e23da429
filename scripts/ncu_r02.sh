#!/bin/bash
# ncu --set full of one steady-state launch of each hot kernel at the bench config.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1 RGBDSEG_B200_AUTOBUILD=0
for ks in ${KERNELS:-gmm_step:12 pbas_classify_strip:200 pbas_apply_list:350}; do
  k=${ks%%:*}; skip=${ks##*:}
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
    -o gpurun_out/full_$k python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-verify \
    > gpurun_out/full_$k.log 2>&1
  echo "$k rc=$?"
done

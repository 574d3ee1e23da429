#!/bin/bash
# ncu --set full of ONE steady-state launch of the kernels named in $KERNELS
# (regex:skip pairs) at the bench's own configuration; reports -> gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for ks in ${KERNELS:-pbas_classify:45}; do
  k=${ks%%:*}; skip=${ks##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
    -o gpurun_out/full_${TAG:-x}_$k python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
    ${BENCH_ARGS} > gpurun_out/full_${TAG:-x}_$k.log 2>&1
  echo "$k rc=$?"
done

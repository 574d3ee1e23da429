#!/bin/bash
# Final evidence: ncu --set full of ONE steady-state launch of each hot kernel
# at the bench's own configuration (8 x 1080p streams), plus the launch list.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo "BUILD FAILED"; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/launches.log 2>&1
# burn-in = 40 frames; the solo phase follows; skip into steady state
for ks in gmm_step:45 pbas_classify:45 pbas_apply_list:25; do
  k=${ks%%:*}; skip=${ks##*:}
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
    -o gpurun_out/full_$k python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/full_$k.log 2>&1
  echo "$k rc=$?"
done
ls -la gpurun_out/*.ncu-rep

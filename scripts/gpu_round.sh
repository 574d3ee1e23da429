#!/bin/bash
# One GPU session: parity tests, a short bench, ncu launch list + full captures.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
{ nvidia-smi; nproc; lscpu | head -20; } > gpurun_out/box.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo "BUILD FAILED"; tail -30 gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout ${PYTEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q -rA ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS:---steps 10 --warmup 3} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
if [ -z "$SKIP_NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/launches.log 2>&1
for ks in gmm_step:44 pbas_classify:44 pbas_apply:22; do
k=${ks%%:*}; skip=${ks##*:}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
  -o gpurun_out/prof_$k python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --streams 1 \
  > gpurun_out/ncu_$k.log 2>&1
done
fi
ls -la gpurun_out

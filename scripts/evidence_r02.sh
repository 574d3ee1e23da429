#!/bin/bash
# Round-2 evidence pass on one B200 (prebuilt in-tree .so): smoke, GPU tests,
# default bench line, f32 line, reference arm, every BASELINE config line,
# launch list and ncu --set full of the hot kernels at the bench config.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1 RGBDSEG_B200_AUTOBUILD=0
{ nvidia-smi; nproc; } > gpurun_out/box.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rA --timeout 600 --timeout-method thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --gmm-state f32 --no-verify > gpurun_out/bench_gmm_f32.json 2> gpurun_out/bench_gmm_f32.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
[ -z "$SKIP_CONFIGS" ] && CONFIG_ARGS="--no-verify" bash scripts/configs.sh > gpurun_out/configs.txt 2>&1
if [ -z "$SKIP_NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-verify \
    > gpurun_out/launches.log 2>&1
  # GMM: 8 burn-in + solo; PBAS: strips from ~frame 150 of the 400-frame ageing, K3 list at steady state
  # the strip K2 at T = t_lower from the pinned-variant micro (frame ~450)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:pbas_classify_strip -s 430 -c 1 \
    -o gpurun_out/full_pbas_classify_strip python scripts/micro/pbas_t2_time.py 2 > gpurun_out/full_strip.log 2>&1
  for ks in gmm_step:12 pbas_apply_list:350; do
    k=${ks%%:*}; skip=${ks##*:}
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 \
      -o gpurun_out/full_$k python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-verify \
      > gpurun_out/full_$k.log 2>&1
    echo "$k rc=$?"
  done
fi
ls -la gpurun_out

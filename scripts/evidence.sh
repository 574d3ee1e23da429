#!/bin/bash
# Full evidence pass on one B200: build, smoke, GPU tests, default bench
# line, reference arm, every BASELINE config line, launch list and ncu
# --set full captures of the three hot kernels at the bench configuration.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
{ nvidia-smi; nproc; } > gpurun_out/box.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo "BUILD FAILED"; tail -30 gpurun_out/build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --gmm-state f32 > gpurun_out/bench_gmm_f32.json 2> gpurun_out/bench_gmm_f32.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
[ -z "$SKIP_CONFIGS" ] && bash scripts/configs.sh > gpurun_out/configs.txt 2>&1
[ -z "$SKIP_NCU" ] && bash scripts/ncu_evidence.sh > gpurun_out/ncu_evidence.txt 2>&1
ls -la gpurun_out

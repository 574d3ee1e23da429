#!/bin/bash
# f32 GMM storage: GPU tests, bench A/B (f64 default vs --gmm-state f32), one ncu capture.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gmm_f32.py tests/test_gpu_parity.py -m gpu -q -x -k "gmm or f32 or golden" > gpurun_out/pytest_f32.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f32.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_f64.json 2> gpurun_out/bench_f64.err
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --gmm-state f32 > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gmm_step -s 44 -c 1 \
    -o gpurun_out/full_f32_gmm python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --gmm-state f32 > gpurun_out/full_f32_gmm.log 2>&1
echo done

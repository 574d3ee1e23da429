cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for wl in config1 config2; do for fl in write write+read; do
  timeout 300 python bench.py --workload $wl --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --flush $fl > gpurun_out/f_${wl}_${fl}.json 2>gpurun_out/f_${wl}.err
done; done
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_clk.json 2>gpurun_out/bench_clk.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch_c2.csv python bench.py --workload config2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch_c1.csv python bench.py --workload config1 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1

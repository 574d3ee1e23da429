#!/bin/bash
# Copy the outputs of scripts/evidence.sh (gpurun_out/) into profiles/r01/.
cd "$(dirname "$0")/.."
P=profiles/r01
cp gpurun_out/bench.json $P/final_bench.json
cp gpurun_out/bench_ref.json $P/final_bench_ref.json
cp gpurun_out/bench_gmm_f32.json $P/final_bench_gmm_f32.json
for c in 1 2 3 4 5; do cp gpurun_out/cfg_config$c.json $P/configs/cfg_config$c.json; done
cp gpurun_out/cfg_config5.json $P/final_bench_c5.json
cp gpurun_out/launches.csv $P/launches_final.csv
for k in gmm_step pbas_classify pbas_apply_list; do cp gpurun_out/full_$k.ncu-rep $P/ncu/full_$k.ncu-rep; done
cp gpurun_out/pytest_gpu.log $P/pytest_gpu_final.log
python scripts/traffic_json.py profiles/traffic.json gmm:config4=$P/ncu/full_gmm_step.ncu-rep \
  pbas:config4=$P/ncu/full_pbas_classify.ncu-rep pbas_apply:config4=$P/ncu/full_pbas_apply_list.ncu-rep
{ python scripts/ncu_summary.py /dev/stdout $P/ncu/full_gmm_step.ncu-rep $P/ncu/full_pbas_classify.ncu-rep \
    $P/ncu/full_pbas_apply_list.ncu-rep 2>/dev/null | head -5
  echo "### gmm_step"; python scripts/ncu_stalls.py $P/ncu/full_gmm_step.ncu-rep
  echo "### pbas_classify"; python scripts/ncu_stalls.py $P/ncu/full_pbas_classify.ncu-rep
  echo
  echo 'Captures: `profiles/r01/ncu/full_*.ncu-rep` -- `ncu --set full --clock-control none` of one steady-state launch of each kernel at the bench configuration (8 x 1920x1080 streams per launch; `scripts/ncu_evidence.sh`). DRAM bytes per launch in `profiles/traffic.json`. Per-launch times from the launch list of the same bench command: `launches_final.csv` (`scripts/launch_times.py`).'
} > $P/ncu_final_summary.md
python scripts/launch_times.py $P/launches_final.csv | head -4

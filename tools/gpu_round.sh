#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full capture of one
# bench step (tools/profile_step.py with the bench's tuned schedules).
# Outputs land in gpurun_out/; tools/ncu_summary.py turns them into profiles/.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/ -q -m gpu 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 120 python tools/pcie_probe.py --bench gpurun_out/bench.json > gpurun_out/pcie.json 2>&1
timeout 600 python tools/cpu_configs.py --bench gpurun_out/bench.json --out gpurun_out/cpu_configs.json > gpurun_out/cpu_configs.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:alcop --csv --log-file gpurun_out/launches.csv \
    python tools/profile_step.py --bench gpurun_out/bench.json --steps 24 > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:alcop -s 8 -c 4 \
    -o gpurun_out/prof_step -f python tools/profile_step.py --bench gpurun_out/bench.json --steps 3 > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/prof_step.ncu-rep --page raw --csv > gpurun_out/prof_step_raw.csv 2>/dev/null
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; cat gpurun_out/pcie.json; head -c 1500 gpurun_out/bench.json

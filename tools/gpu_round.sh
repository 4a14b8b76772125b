#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full capture of the
# dominant bench kernel.  Outputs land in gpurun_out/.
set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/ -q -m gpu 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:alcop -s 60 -c 60 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 5 --quick --no-cpu > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:alcop -s 64 -c 2 \
    -o gpurun_out/prof_bench python bench.py --steps 20 --warmup 5 --quick --no-cpu > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; cat gpurun_out/bench.json | head -c 3000

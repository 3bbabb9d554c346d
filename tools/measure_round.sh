#!/bin/bash
# Round measurement on one B200 (run under gpurun): GPU tests, bench line,
# C5 sweep, C2 convergence, launch list and ncu captures of the headline kernels.
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/m_tests.log 2>&1
timeout 600 python bench.py > gpurun_out/m_bench.log 2>&1
timeout 1200 python tools/sweep.py --out gpurun_out/m_sweep.jsonl > gpurun_out/m_sweep.log 2>&1
timeout 300 python tools/c2_converge.py --out gpurun_out/m_converge.md > /dev/null 2>&1
timeout 600 python tools/cum_bench.py --out gpurun_out/m_cum.jsonl > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/m_launches_c4.csv python bench.py --steps 1 --warmup 3 --secondary '' --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lane_ps3g -c 1 -o gpurun_out/m_c4_full python tools/ncu_target.py --workload c4 --slices 2000 --repeat 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lane_ps_kernel -c 1 -o gpurun_out/m_c3_full python tools/ncu_target.py --workload c3 --slices 20000 --repeat 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lane_small -c 1 -o gpurun_out/m_c1m_full python tools/ncu_qubit.py 1000000 > /dev/null 2>&1
tail -2 gpurun_out/m_tests.log

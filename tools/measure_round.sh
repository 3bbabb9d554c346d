#!/bin/bash
# Round measurement on one B200 (run under gpurun): GPU tests, bench line,
# full-size DRAM traffic of the headline kernels, launch list, ncu --set full
# captures of the C4, c1m (su2) and D64 lane kernels.  Outputs: gpurun_out/m_*.
set -x
P=${1:-m}
# full-size DRAM traffic first: a fresh process on a fresh box (the L2 state left by
# earlier processes changes the write-back / re-read traffic of the exchange buffers)
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:lane_ps3g -c 1 --csv --log-file gpurun_out/${P}_traffic_c4.csv python tools/ncu_target.py --workload c4 --slices 1000000 --repeat 1 > /dev/null 2>&1
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:lane_su2 -c 1 --csv --log-file gpurun_out/${P}_traffic_c1m.csv python tools/ncu_target.py --workload c1m --slices 1000000 --repeat 1 > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/${P}_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/${P}_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${P}_launches_c4.csv python bench.py --steps 1 --warmup 3 --secondary '' --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lane_ps3g -c 1 -o gpurun_out/${P}_c4_full python tools/ncu_target.py --workload c4 --slices 2000 --repeat 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lane_su2 -c 1 -o gpurun_out/${P}_c1m_full python tools/ncu_target.py --workload c1m --slices 1000000 --repeat 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:lane_ps3g -c 1 -o gpurun_out/${P}_d64_full python tools/env_ab_target.py 64 2 20000 > /dev/null 2>&1
# summaries on the box; the .ncu-rep files stay there (gpurun copies back <= 64 MiB)
python tools/ncu_summary.py full gpurun_out/${P}_c4_full.ncu-rep "# ncu --set full -k regex:lane_ps3g -c 1 tools/ncu_target.py --workload c4 --slices 2000" > gpurun_out/${P}_ncu_c4.txt 2>&1
python tools/ncu_summary.py full gpurun_out/${P}_c1m_full.ncu-rep "# ncu --set full -k regex:lane_su2 -c 1 tools/ncu_target.py --workload c1m --slices 1000000" > gpurun_out/${P}_ncu_c1m.txt 2>&1
python tools/ncu_summary.py full gpurun_out/${P}_d64_full.ncu-rep "# ncu --set full -k regex:lane_ps3g -c 1 tools/env_ab_target.py 64 2 20000" > gpurun_out/${P}_ncu_d64.txt 2>&1
python tools/ncu_summary.py launches gpurun_out/${P}_launches_c4.csv "# ncu --metrics gpu__time_duration.sum bench.py --steps 1 --warmup 3 (C4 headline)" > gpurun_out/${P}_launches_c4.txt 2>&1
rm -f gpurun_out/${P}_*.ncu-rep
tail -3 gpurun_out/${P}_tests.log

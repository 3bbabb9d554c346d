set -x
timeout 600 python bench.py > gpurun_out/bench_r1c.log 2>&1
timeout 1200 python tools/sweep.py --out gpurun_out/sweep_r1c.jsonl > gpurun_out/sweep_r1c.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 3 --secondary '' --no-cpu > gpurun_out/launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lane_ps3g -c 1 -o gpurun_out/c4_full python tools/ncu_target.py --workload c4 --slices 2000 --repeat 1 > gpurun_out/c4_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lane_ps_kernel -c 1 -o gpurun_out/c3_full python tools/ncu_target.py --workload c3 --slices 20000 --repeat 1 > gpurun_out/c3_full.log 2>&1
ls -la gpurun_out

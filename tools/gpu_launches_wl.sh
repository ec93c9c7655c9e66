#!/bin/bash
# ncu launch list (durations only) of one bench workload: bash tools/gpu_launches_wl.sh cfg4
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/prof
wl=${1:-cfg4}
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_$wl.csv \
   python bench.py --workload $wl --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/prof/b_ncu_$wl.log 2>&1
echo "rc=$?"
python tools/launch_summary.py gpurun_out/prof/launches_$wl.csv 5 > gpurun_out/prof/launches_$wl.txt 2>&1
head -30 gpurun_out/prof/launches_$wl.txt

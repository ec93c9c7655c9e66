#!/bin/bash
# Final round-2 evidence pass on one B200: launch list of the default bench
# (ncu duration-only, cold serialised), the ncu summaries of every workload's
# search kernel and of the cfg3 index kernels (gpu_prof_r2.sh).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/prof
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv \
   python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/prof/b_ncu.log 2>&1
echo "launches rc=$?"
python tools/launch_summary.py gpurun_out/prof/launches.csv 5 > gpurun_out/prof/launches_cfg3.txt 2>&1
bash tools/gpu_prof_r2.sh "$@"

#!/bin/bash
# per-kernel launch times of quick_time ticks: bash tools/gpu_launches.sh [dist n nq k] > gpurun_out/launch_summary.txt
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
QT_ITERS=3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_qt.csv python tools/quick_time.py ${1:-gaussian} ${2:-1e7} ${3:-1e6} ${4:-32} > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_qt.csv 4

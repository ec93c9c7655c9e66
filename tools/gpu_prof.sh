#!/bin/bash
# ncu pass: launch list + full capture of the search kernel ($1 = extra bench args)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline $1 > gpurun_out/b_ncu.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_search -s 2 -c 1 \
   -o gpurun_out/search_full -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline $1 > gpurun_out/b_ncufull.log 2>&1
tail -2 gpurun_out/b_ncufull.log

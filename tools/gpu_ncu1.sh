#!/bin/bash
# full ncu capture of the k<=32 search kernel on one workload: $1 tag, $2.. ab_search args
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=$1; shift
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_search -s 2 -c 1 \
   -o gpurun_out/search_$tag -f python tools/ab_search.py "$@" 3 > gpurun_out/ncu_$tag.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_$tag.log

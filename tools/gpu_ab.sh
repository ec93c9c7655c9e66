#!/bin/bash
# A/B of the search kernels: v1 (positions lists, direct loads), v1+TMA ring,
# v0 (MKNN_SEARCH_V0=1); $1 = tag, $2 = "prof" to add a work-counter build pass
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=${1:-ab}
WLS=${WLS:-"gaussian 1e7 1e6 32|uniform 1e7 1e6 32|uniform 1e6 1e5 32"}
IFS='|' read -ra wls <<< "$WLS"
for wl in "${wls[@]}"; do
  for v in ${VARS:-0 2}; do
    MKNN_SEARCH_VAR=$v timeout 300 python tools/ab_search.py $wl 2>&1 | tail -1 | sed "s/^v1/var$v/"
  done
  MKNN_SEARCH_V0=1 timeout 300 python tools/ab_search.py $wl 2>&1 | tail -1
done | tee gpurun_out/ab_$tag.txt
if [ "$2" = "prof" ]; then
  (cd paper_1412_6170_b200/csrc && make -s clean && make -s -j8 EXTRA=-DMKNN_PROFILE=1 > /dev/null 2>&1)
  for v in 0 1; do
    MKNN_SEARCH_V0=$([ $v = 0 ] && echo 1 || echo 0) MKNN_PROF=1 timeout 300 python tools/ab_search.py gaussian 1e7 1e6 32 2 2>&1 | grep "mknn prof" | tail -1
  done | tee -a gpurun_out/ab_$tag.txt
fi

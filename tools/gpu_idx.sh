#!/bin/bash
# re-index variants (env combos) on cfg3 and uniform 10M; $1 tag
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for combo in "X=0" "MKNN_SCATTER=1" "MKNN_SUBCELL=16" "MKNN_SCATTER=1 MKNN_SUBCELL=16" "MKNN_SUBCELL=8" "MKNN_SCATTER=1 MKNN_SUBCELL=8"; do
  for wl in "gaussian 1e7 1e6 32" "uniform 1e7 1e6 32"; do
    env $combo AB_TAG="[$combo]" timeout 300 python tools/ab_search.py $wl 2>&1 | tail -1
  done
done | tee gpurun_out/idx_$1.txt

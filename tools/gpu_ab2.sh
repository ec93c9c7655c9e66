#!/bin/bash
# A/B of env-switched variants: VARS="ENV=a ENV=b ..." over WLS workloads; then
# (optional, $2 = tests) the GPU parity tests. $1 = tag.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=${1:-ab}
WLS=${WLS:-"gaussian 1e7 1e6 32|uniform 1e7 1e6 32|uniform 1e6 1e5 32"}
IFS='|' read -ra wls <<< "$WLS"
for wl in "${wls[@]}"; do
  for v in ${VARS:-X=0}; do
    env $v AB_TAG="[$v]" timeout 300 python tools/ab_search.py $wl 2>&1 | tail -1
  done
done | tee gpurun_out/ab_$tag.txt
if [ "$2" = "tests" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q ${TESTS:-} > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
  tail -3 gpurun_out/pytest_$tag.log
fi

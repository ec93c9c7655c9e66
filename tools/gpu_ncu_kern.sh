#!/bin/bash
# ncu --set full of the kernels matching $2 on tools/ab_search.py $3.. (one
# launch each after $1 skips), summarised on the box: gpurun_out/ncu_$TAG.txt
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
skip=$1; regex=$2; shift 2
tag=${TAG:-kern}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$regex" -s $skip -c ${COUNT:-2} \
  -o /tmp/ncu_$tag -f python tools/ab_search.py "$@" 2 > gpurun_out/ncu_$tag.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py /tmp/ncu_$tag.ncu-rep > gpurun_out/ncu_$tag.txt 2>&1
if [ -n "$SRC" ]; then
  ncu -i /tmp/ncu_$tag.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_$tag.csv 2>/dev/null
  python tools/ncu_lines.py /tmp/src_$tag.csv 40 >> gpurun_out/ncu_$tag.txt 2>&1
fi

#!/bin/bash
# copy the gpu_round.sh + gpu_matrix.sh outputs into profiles/ as version $1 (e.g. v6)
set -e
cd /root/repo
v=$1
for wl in cfg2 cfg3 cfg3u k1 k8 k32 k128 cfg4; do cp gpurun_out/matrix/$wl.json profiles/r1_bench_${wl}_$v.json; done
cp gpurun_out/bench.json profiles/r1_bench_default_$v.json
python tools/launch_summary.py gpurun_out/launches.csv 5 > profiles/r1_launches_cfg3_$v.txt 2>/dev/null || true
ncu -i gpurun_out/search_full.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_$v.csv 2>/dev/null
(python tools/ncu_summary.py gpurun_out/search_full.ncu-rep; echo; echo "# per-function share"; \
 python tools/ncu_funcs.py /tmp/src_$v.csv | head -25; echo; echo "# top stall lines"; \
 python tools/ncu_lines.py /tmp/src_$v.csv 20 | tail -20) > profiles/r1_search_ncu_$v.txt 2>&1
head -16 profiles/r1_search_ncu_$v.txt

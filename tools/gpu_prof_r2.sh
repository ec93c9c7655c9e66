#!/bin/bash
# Round-2 ncu pass: one full capture of the search kernel per BASELINE workload
# and of the cfg3 index kernels, summarised on the box (gpurun_out/prof/*.txt;
# only the cfg3 search capture is kept as a .ncu-rep). $@ = workloads.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/prof
P=gpurun_out/prof
for wl in ${@:-cfg3 cfg3u cfg2 k1 k8 k128 cfg4}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_search -s 2 -c 1 \
    -o $P/search_$wl -f python bench.py --workload $wl --steps 1 --warmup 3 --e2e-steps 0 \
    --no-cpu-baseline > $P/search_$wl.log 2>&1
  echo "$wl rc=$?"
  python tools/ncu_summary.py $P/search_$wl.ncu-rep > $P/search_$wl.txt 2>&1
  ncu -i $P/search_$wl.ncu-rep --page source --csv --print-source cuda,sass > /tmp/src_$wl.csv 2>/dev/null
  (echo "# per-function share"; python tools/ncu_funcs.py /tmp/src_$wl.csv | head -30; echo; echo "# top lines"; \
   python tools/ncu_lines.py /tmp/src_$wl.csv 40) >> $P/search_$wl.txt 2>&1
  [ "$wl" = "cfg3" ] || rm -f $P/search_$wl.ncu-rep
done
timeout 900 ncu --set full --clock-control none \
  -k regex:"k_point_keys|k_partition|k_final_scatter|k_chunk_boxes|k_scan|k_bucket|k_leaf_ranges|k_chunk_ranges|k_q_scatter|k_issuer" \
  -s 40 -c 30 -o $P/index_cfg3 -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 \
  --no-cpu-baseline > $P/index_cfg3.log 2>&1
echo "index rc=$?"
python tools/ncu_summary.py $P/index_cfg3.ncu-rep > $P/index_cfg3.txt 2>&1
rm -f $P/index_cfg3.ncu-rep
du -sh gpurun_out

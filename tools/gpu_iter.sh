#!/bin/bash
# Iteration pass: gpu tests (stop at first failure), bench line, full ncu of the search kernel.
# $1: tag for the output files; $2: "notest" to skip pytest
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=${1:-it}
if [ "$2" != "notest" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
  tail -14 gpurun_out/pytest_$tag.log
fi
timeout 600 python bench.py --steps 10 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
python -c "import json;d=json.load(open('gpurun_out/bench_$tag.json'));print(round(d['value']/1e6,2),'Mq/s',round(d['ms_per_step'],3),'ms',d['tick_phases_us'],'e2e',round(d['e2e']['value']/1e6,2))" || tail -5 gpurun_out/bench_$tag.err
MKNN_PROF=1 timeout 300 python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline > /dev/null 2> gpurun_out/prof_$tag.err
grep "mknn prof" gpurun_out/prof_$tag.err | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_search -s 2 -c 1 \
   -o gpurun_out/search_$tag -f python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1
echo "ncu rc=$?"

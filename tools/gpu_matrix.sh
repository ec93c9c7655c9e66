#!/bin/bash
# bench.py over every BASELINE.json workload (1 GPU): gpurun_out/matrix/<workload>.json
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/matrix
for wl in ${@:-cfg2 cfg3 cfg3u k1 k8 k32 k128 cfg4}; do
  extra="--no-cpu-baseline"
  [ "$wl" = "cfg2" ] && extra=""
  timeout 900 python bench.py --workload $wl --steps 10 --warmup 3 --e2e-steps 2 $extra \
    > gpurun_out/matrix/$wl.json 2> gpurun_out/matrix/$wl.err
  echo "$wl rc=$? $(python -c "import json;d=json.load(open('gpurun_out/matrix/$wl.json'));print(round(d['value']/1e6,2),'Mq/s',round(d['ms_per_step'],3),'ms',d['tick_phases_us'])" 2>&1 | tail -1)"
done

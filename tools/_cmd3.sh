mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_fuse.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fuse.log; tail -2 gpurun_out/pytest_fuse.log
WLS="gaussian 1e7 1e6 32|uniform 1e7 1e6 32|uniform 1e6 1e5 32" VARS="MKNN_BSORT=0 MKNN_BSORT=1" bash tools/gpu_ab2.sh fuse
python tools/graph_probe.py 2>&1 | tail -3
timeout 900 python bench.py --steps 10 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err
python -c "import json;d=json.load(open('gpurun_out/bench_f.json'));print(d['value']/1e6, d['ms_per_step'], d['e2e']['value']/1e6, d['tick_phases_us'])"
timeout 900 python bench.py --workload cfg2 --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_f2.json 2> gpurun_out/bench_f2.err
python -c "import json;d=json.load(open('gpurun_out/bench_f2.json'));print(d['value']/1e6, d['ms_per_step'], d['e2e']['value']/1e6, d['tick_phases_us'])"

mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
bash tools/gpu_matrix.sh cfg2 cfg3 cfg3u k1 k8 k32 k128 cfg4 > gpurun_out/matrix.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --e2e-steps 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 1200 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 3 > gpurun_out/launches_cfg3.txt 2>&1
bash tools/gpu_prof_r2.sh cfg3 cfg3u cfg2 k1 k8 k128 cfg4 > gpurun_out/prof.txt 2>&1

mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/pytest_r2c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2c.log
tail -12 gpurun_out/pytest_r2c.log
for wl in cfg2 cfg3; do
  timeout 600 python bench.py --workload $wl --steps 20 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bg_$wl.json 2> gpurun_out/bg_$wl.err
done

timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_upd.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_upd.log; tail -2 gpurun_out/pytest_upd.log
for wl in cfg2 cfg4; do
  timeout 900 python bench.py --workload $wl --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bu_$wl.json 2> gpurun_out/bu_$wl.err
done

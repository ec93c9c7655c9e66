for cfg in "MKNN_H2D_OVERLAP=0" "MKNN_H2D_OVERLAP=1" "MKNN_H2D_OVERLAP=0" "MKNN_H2D_OVERLAP=1"; do
  env $cfg timeout 600 python bench.py --steps 2 --warmup 3 --e2e-steps 6 --no-cpu-baseline > gpurun_out/bov.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bov.json'));print('$cfg', round(d['value']/1e6,1), round(d['e2e']['value']/1e6,2))"
done
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_ov.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ov.log; tail -2 gpurun_out/pytest_ov.log

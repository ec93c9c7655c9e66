#!/bin/bash
# A/B of compile-time variants (variants/<name>/libmknn_b200.so, tools/build_variant.sh)
# against the default library. LIBS="base name1 name2", WLS as in gpu_ab2.sh; $1 = tag;
# $2 = tests: then the GPU parity suite on the default library.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=${1:-ablib}
IFS='|' read -ra wls <<< "${WLS:-gaussian 1e7 1e6 128}"
for wl in "${wls[@]}"; do
  for v in ${LIBS:-base}; do
    if [ "$v" = base ]; then lib=""; else lib=variants/$v/libmknn_b200.so; fi
    MKNN_LIB=$lib AB_TAG="[$v]" timeout 300 python tools/ab_search.py $wl 2>&1 | tail -1
  done
done | tee gpurun_out/ab_$tag.txt
if [ "$2" = "tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q ${TESTS:-} > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
  tail -3 gpurun_out/pytest_$tag.log
fi

#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_case.py
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
out=gpurun_out/sanitizer.txt; : > $out
for tool in memcheck racecheck synccheck; do
  echo "== compute-sanitizer --tool $tool python tools/sanitize_case.py" >> $out
  timeout 1500 compute-sanitizer --tool $tool python tools/sanitize_case.py >> $out 2>&1
  echo "rc=$?" >> $out
done
grep -E "SUMMARY|rc=" $out

#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the round-2 kernels
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
OUT=gpurun_out/r02_sanitizer.txt
: > $OUT
for script in sanitize_tc sanitize_mem; do
  echo "# compute-sanitizer: scripts/$script.py" >> $OUT
  for tool in memcheck racecheck synccheck; do
    echo "## $tool" >> $OUT
    timeout 1200 compute-sanitizer --tool $tool python scripts/$script.py 2>&1 | grep -E "^ok|SUMMARY|Error|error" | head -20 >> $OUT
    echo "rc=${PIPESTATUS[0]}" >> $OUT
  done
done
echo done

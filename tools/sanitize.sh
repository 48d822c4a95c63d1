#!/bin/bash
# compute-sanitizer over the smoke invocation (one tool per gpurun call: the
# B200 profiling guide warns against running several tools in one call).
# usage: tools/sanitize.sh memcheck|racecheck|synccheck|initcheck
tool=${1:-memcheck}
mkdir -p gpurun_out
extra=""
[ "$tool" = "memcheck" ] && extra="--leak-check no"
timeout 1500 compute-sanitizer --tool "$tool" $extra --print-limit 50 --error-exitcode 9 \
  python -c "import __graft_entry__ as g; g.smoke()" > "gpurun_out/sanitize_$tool.log" 2>&1
echo "exit $?" >> "gpurun_out/sanitize_$tool.log"
tail -5 "gpurun_out/sanitize_$tool.log"

# compute-sanitizer over tools/sanitize_cases.py, ONE tool per invocation (run each in its own
# gpurun call: B200_PROFILING.md reports a GPU left unusable after several tools in one call).
#   /usr/local/graft/bin/gpurun -- 'bash tools/sanitize.sh memcheck'   (then racecheck, synccheck)
set -u
tool=${1:-memcheck}
mkdir -p gpurun_out
python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/sanitize_plain.log; exit 1; }
timeout 1500 compute-sanitizer --tool "$tool" --error-exitcode 9 --print-limit 50 python tools/sanitize_cases.py \
    > gpurun_out/sanitize_$tool.log 2>&1
echo "$tool exit $?"; tail -5 gpurun_out/sanitize_$tool.log

# compute-sanitizer on the small persistent-sweep case (one tool per call of
# this script: TOOL=racecheck|memcheck|synccheck)
mkdir -p gpurun_out
TOOL=${TOOL:-racecheck}
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitizer_case.py > gpurun_out/r2_sanitize_$TOOL.txt 2>&1
echo "rc=$?" >> gpurun_out/r2_sanitize_$TOOL.txt

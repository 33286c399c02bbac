# r02: compute-sanitizer memcheck / racecheck / synccheck over the production kernels
set -x
O=gpurun_out/r02j; mkdir -p $O
python tools/prof/sanitize.py > $O/plain.log 2>&1; echo plain rc=$?; tail -2 $O/plain.log
for tool in memcheck racecheck synccheck; do
  ZKL_FORCE_PERSISTENT=1 timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/prof/sanitize.py > $O/$tool.log 2>&1; echo $tool rc=$?; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok |complete|Error|error" $O/$tool.log | tail -14
done

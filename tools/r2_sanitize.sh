# compute-sanitizer memcheck / racecheck / synccheck over every kernel (tools/sanitize_smoke.py)
set -u
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_smoke.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitize_$tool.txt
done

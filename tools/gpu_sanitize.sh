# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_drive.py
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_drive.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -n 4 gpurun_out/sanitize_$tool.log
done

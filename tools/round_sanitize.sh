# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize.py (every kernel family, small sizes)
T=${1:-r02}
for tool in memcheck racecheck synccheck; do
  echo "### compute-sanitizer --tool $tool python tools/sanitize.py" >> gpurun_out/${T}_sanitizer.txt
  timeout 1500 compute-sanitizer --tool $tool --print-limit 200 python tools/sanitize.py > gpurun_out/${T}_san_$tool.log 2>&1
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Race reported|and (Read|Write) access|^ok" gpurun_out/${T}_san_$tool.log | sort | uniq -c >> gpurun_out/${T}_sanitizer.txt
done

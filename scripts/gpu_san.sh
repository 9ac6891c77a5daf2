O=gpurun_out/${TAG:-san}
mkdir -p $O
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_run.py > $O/sanitizer_$tool.log 2>&1; echo "rc=$?" >> $O/sanitizer_$tool.log
done

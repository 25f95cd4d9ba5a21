mkdir -p gpurun_out
OUT=gpurun_out/r2_sanitizers.txt
echo "# compute-sanitizer over scripts/sanitize_cases.py (smoke() + k = 2 in-epilogue combine + fp32 accumulate), B200, round 2" > $OUT
for tool in memcheck synccheck racecheck; do
  echo "## $tool" >> $OUT
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/san_$tool.log 2>&1; echo "rc=$?" >> $OUT
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error:|Race reported|case |smoke" gpurun_out/san_$tool.log | sort | uniq -c | sort -rn | head -25 >> $OUT
done
cat $OUT

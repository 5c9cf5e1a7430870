# compute-sanitizer over tests/sanitize_cases.py (every tool), summary to gpurun_out/sanitizer.txt
O=gpurun_out/sanitizer.txt
echo "== compute-sanitizer over tests/sanitize_cases.py (B200, round 2 late: + the cp.async-ring x histogram, shared-typed tile scratch, 128-row TMA boxes in the MIN/MAX one pass)" > $O
for tool in memcheck racecheck synccheck initcheck; do
  echo "== compute-sanitizer --tool $tool python tests/sanitize_cases.py" >> $O
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $tool python tests/sanitize_cases.py > /tmp/san_$tool.txt 2>&1; grep -E "COMPUTE-SANITIZER|SUMMARY|done|Error|error|Hazard|hazard" /tmp/san_$tool.txt | head -40 >> $O; tail -3 /tmp/san_$tool.txt >> $O
done

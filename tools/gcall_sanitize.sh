# compute-sanitizer over tests/sanitize_cases.py (every tool), summary to gpurun_out/sanitizer.txt
O=gpurun_out/sanitizer.txt
echo "== compute-sanitizer over tests/sanitize_cases.py (B200, round 2 late: + the warp-specialised scan_reduce (named barriers), the cp.async-ring x histogram, shared-typed tile scratch)" > $O
for tool in memcheck racecheck synccheck initcheck; do
  echo "== compute-sanitizer --tool $tool python tests/sanitize_cases.py" >> $O
  timeout 1200 compute-sanitizer --tool $tool python tests/sanitize_cases.py 2>&1 | grep -E "COMPUTE-SANITIZER|SUMMARY|done|Error|error|Hazard|hazard" | head -40 >> $O
done

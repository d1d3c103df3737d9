# compute-sanitizer tiers over tools/sanitize.py (run under gpurun).
for T in memcheck racecheck synccheck; do
  echo "== $T"
  timeout 1200 compute-sanitizer --tool $T --print-limit 20 python tools/sanitize.py 2>&1 | grep -E "SUMMARY|loss|Error|error" | head -30
done

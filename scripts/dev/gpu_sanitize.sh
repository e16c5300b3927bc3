for tool in memcheck racecheck synccheck; do
  echo "== $tool"; timeout 900 compute-sanitizer --tool $tool --print-limit 5 python scripts/dev/sanitize_r02.py 2>&1 | grep -E "ERROR SUMMARY|Error|error|channel-sharded" | head -8
done

cd /root/repo
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py 2>&1 | grep -vE "^$" | tail -15
done

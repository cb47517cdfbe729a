# compute-sanitizer over every kernel family (tools/sanitize_cases.py) on the shipped build
O=gpurun_out/sanitize
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool "$tool" python tools/sanitize_cases.py > "$O/$tool.log" 2>&1
  echo "$tool rc=$?" >> "$O/summary.txt"
  tail -2 "$O/$tool.log" >> "$O/summary.txt"
done

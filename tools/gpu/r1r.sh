set -x
O=gpurun_out/r1r
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/sanitize_cases.py > $O/plain.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_cases.py > $O/memcheck.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python tools/sanitize_cases.py > $O/racecheck.log 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_cases.py > $O/synccheck.log 2>&1
timeout 900 compute-sanitizer --tool initcheck --print-limit 20 python tools/sanitize_cases.py > $O/initcheck.log 2>&1
ls -la $O

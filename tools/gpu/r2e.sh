set -x
O=gpurun_out/r2e
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_cases.py > $O/memcheck.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python tools/sanitize_cases.py > $O/racecheck.log 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_cases.py > $O/synccheck.log 2>&1
ls -la $O

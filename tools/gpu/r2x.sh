set -x
O=gpurun_out/r2x
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "products or c1_goldens or c2_scale or c3_scale or pair_kernel or randomized" > $O/pytest.log 2>&1
timeout 600 python bench.py --no-cpu --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config c3 --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 10 python tools/sanitize_cases.py > $O/racecheck.log 2>&1
ls -la $O

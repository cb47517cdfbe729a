set -x
O=gpurun_out/r1y
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --config c3 --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python tools/sweep_bench.py > $O/sweep_default.json 2> $O/sweep_default.err
ls -la $O

set -x
O=gpurun_out/r2y
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1800 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py --no-cpu --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
ls -la $O

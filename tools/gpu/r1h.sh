set -x
O=gpurun_out/r1h
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_engine.py -x -q > $O/pytest_engine.log 2>&1
timeout 600 python tools/service_bench.py > $O/service_c2.json 2> $O/service_c2.err
ls -la $O

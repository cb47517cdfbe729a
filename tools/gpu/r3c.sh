set -x
O=gpurun_out/r3c
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "native_pipeline or sharded" > $O/pytest.log 2>&1
timeout 300 python tools/host_overhead.py > $O/host.json 2>&1
timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -x -q -k native_pipeline > $O/memcheck.log 2>&1
ls -la $O

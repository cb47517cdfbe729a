set -x
O=gpurun_out/r1s
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_banded.py tests/test_gpu_engine.py -x -q > $O/pytest.log 2>&1
ls -la $O

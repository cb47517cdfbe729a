set -x
O=gpurun_out/r1t
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "dual_buffer or sweep_and_transfer" > $O/pytest.log 2>&1
timeout 900 python tools/dual_bench.py > $O/dual.json 2> $O/dual.err
ls -la $O

set -x
O=gpurun_out/r2g
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gram or products or c3_scale or c2_scale" > $O/pytest.log 2>&1
timeout 900 python tools/k_sweep.py > $O/k_sweep.jsonl 2> $O/k_sweep.err
ls -la $O

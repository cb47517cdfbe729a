set -x
O=gpurun_out/r2k
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "pair_kernel" > $O/pytest.log 2>&1
timeout 1200 python tools/k_sweep.py > $O/k_sweep.jsonl 2> $O/k_sweep.err
ls -la $O

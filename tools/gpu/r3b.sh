set -x
O=gpurun_out/r3b
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gram or products or randomized or pair_kernel" > $O/pytest.log 2>&1
timeout 900 python tools/k_sweep.py > $O/k_sweep.jsonl 2> $O/k_sweep.err
timeout 600 python -m pytest tests/test_reference_suite_gpu.py -q > $O/pytest_ref.log 2>&1
ls -la $O

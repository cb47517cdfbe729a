set -x
O=gpurun_out/r1i
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "pair_kernel or gram_engines_exact or products_match" > $O/pytest_pair.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c3_scale" > $O/pytest_c3.log 2>&1
timeout 300 python tools/gpu/diag_cap.py > $O/diag_cap.json 2>&1
timeout 600 python bench.py --config c3 --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
ls -la $O

set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r9_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "products" > gpurun_out/r9_pytest_products.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r9_pytest.log 2>&1
timeout 300 python bench.py --no-e2e --no-cpu > gpurun_out/r9_bench.json 2> gpurun_out/r9_bench.err
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_gram_tc -s 3 -c 1 -o gpurun_out/r9_fused python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r9_ncu.log 2>&1

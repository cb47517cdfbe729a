set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r8_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "gram" > gpurun_out/r8_pytest_gram.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r8_pytest.log 2>&1
timeout 300 python bench.py --no-e2e --no-cpu > gpurun_out/r8_bench_f4.json 2> gpurun_out/r8_bench_f4.err
timeout 300 python bench.py --no-e2e --no-cpu --engine tc > gpurun_out/r8_bench_i8.json 2> gpurun_out/r8_bench_i8.err
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_gram_tc -s 2 -c 1 -o gpurun_out/r8_gram python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r8_ncu_gram.log 2>&1

set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r4_build.log 2>&1
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4_smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r4_pytest.log 2>&1
timeout 300 python bench.py --no-e2e --no-cpu > gpurun_out/r4_bench.json 2> gpurun_out/r4_bench.err
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_gram_tc -s 1 -c 1 -o gpurun_out/r4_gram python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r4_ncu_gram.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_overlap -s 1 -c 1 -o gpurun_out/r4_overlap python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r4_ncu_ov.log 2>&1

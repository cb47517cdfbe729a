set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r6_build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r6_pytest.log 2>&1
timeout 300 python bench.py --no-e2e --no-cpu > gpurun_out/r6_bench.json 2> gpurun_out/r6_bench.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_overlap -s 1 -c 1 -o gpurun_out/r6_overlap python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r6_ncu_ov.log 2>&1

set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r7_build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r7_pytest.log 2>&1
timeout 600 python bench.py > gpurun_out/r7_bench.json 2> gpurun_out/r7_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r7_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r7_ncu_bench.log 2>&1

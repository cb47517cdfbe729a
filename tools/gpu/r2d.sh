set -x
O=gpurun_out/r2d
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "device_similarity or sharded" > $O/pytest.log 2>&1
timeout 600 python bench.py --config c3 --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu > $O/ncu_launch_c3.log 2>&1
ls -la $O

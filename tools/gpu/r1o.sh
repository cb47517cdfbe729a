set -x
O=gpurun_out/r1o
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_engine.py -x -q > $O/pytest_engine.log 2>&1
timeout 600 python tools/ingest_bench.py > $O/ingest.json 2> $O/ingest.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu_launch.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_gram_tc -s 2 -c 1 -o $O/recompute_fused python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_fused.log 2>&1
ls -la $O

set -x
O=gpurun_out/r1k
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "pair_kernel or gram_engines_exact or c3_scale" > $O/pytest_pair.log 2>&1
timeout 600 python bench.py --config c3 --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gram_pair -s 1 -c 1 -o $O/gram_pair python bench.py --config c3 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_pair.log 2>&1
ls -la $O

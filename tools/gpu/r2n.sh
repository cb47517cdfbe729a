set -x
O=gpurun_out/r2n
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gram or products or c3_scale or c2_scale or pair_kernel" > $O/pytest.log 2>&1
timeout 600 python bench.py --no-cpu --no-e2e > $O/bench_c2.json 2> $O/bench_c2.err
FS_DIAG_TMA=1 timeout 600 python bench.py --no-cpu --no-e2e > $O/bench_c2_tma.json 2> $O/bench_c2_tma.err
timeout 600 python bench.py --config c3 --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
ls -la $O

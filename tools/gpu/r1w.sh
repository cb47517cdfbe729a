set -x
O=gpurun_out/r1w
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for d in 2 3 4; do
  FS_FUSE_DEPTH=$d timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "products" > $O/pytest_d$d.log 2>&1
  FS_FUSE_DEPTH=$d timeout 600 python bench.py --no-cpu --no-e2e > $O/bench_d$d.json 2> $O/bench_d$d.err
done
ls -la $O

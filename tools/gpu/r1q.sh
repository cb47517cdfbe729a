set -x
O=gpurun_out/r1q
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python bench.py --config c3 --no-cpu --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c1 > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config c1 --impl reference --steps 3 --warmup 1 > $O/bench_c1_reference.json 2> $O/bench_c1_reference.err
ls -la $O

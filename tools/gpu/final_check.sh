# round-end validation on one B200: build, smoke, GPU tests, default bench (C2), the
# reference arm, C1 / C3 benches and a 2-rank (gloo) run of the N>1 bench path
set -x
O=gpurun_out/final3
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$? >> $O/smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py --config c1 > $O/bench_c1.json 2> $O/bench_c1.err
python bench.py --config c3 --no-cpu > $O/bench_c3.json 2> $O/bench_c3.err
FS_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu > $O/bench_n2.json 2> $O/bench_n2.err
python tools/k_sweep.py --fused-only > $O/k_sweep.jsonl 2>&1

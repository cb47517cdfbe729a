set -x
O=gpurun_out/r1u
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
export FS_DIST_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 > $O/bench_n2.json 2> $O/bench_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --impl reference --steps 1 --warmup 0 > $O/bench_n2_ref.json 2> $O/bench_n2_ref.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --config c4 --steps 2 --warmup 1 --max-host-gb 8 > $O/bench_c4_n2.json 2> $O/bench_c4_n2.err
ls -la $O

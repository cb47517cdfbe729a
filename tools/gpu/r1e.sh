set -x
mkdir -p gpurun_out/r1e
O=gpurun_out/r1e
nvidia-smi -q | head -40 > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
ls -la $O

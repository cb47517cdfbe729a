O=gpurun_out/final4
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$? >> $O/smoke.log
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --config c1 > $O/bench_c1.json 2> $O/bench_c1.err
python tools/k_sweep.py --fused-only --cases 16:1024:1024,16:8192:8192,64:8192:8192,128:8192:8192,256:8192:8192,1024:4096:4096 > $O/k_sweep.jsonl 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log

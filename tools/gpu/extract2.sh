mkdir -p gpurun_out/ext2
python -c "import __graft_entry__ as g; g.build()"
python tools/k_sweep.py --cases 16:1024:1024,128:8192:8192,256:8192:8192,1024:4096:4096 > gpurun_out/ext2/ks.jsonl 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/ext2/gpu.log 2>&1; tail -2 gpurun_out/ext2/gpu.log
python bench.py > gpurun_out/ext2/bench_c2.json 2> gpurun_out/ext2/bench_c2.err

mkdir -p gpurun_out/pipe2
python -c "import __graft_entry__ as g; g.build()"
python tools/k_sweep.py --fused-only --cases 256:8192:8192,512:8192:4096,1024:4096:4096,2048:4096:2048 > gpurun_out/pipe2/ks.jsonl 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pipe2/gpu.log 2>&1; tail -2 gpurun_out/pipe2/gpu.log

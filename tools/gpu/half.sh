mkdir -p gpurun_out/half
python -c "import __graft_entry__ as g; g.build()"
python tools/k_sweep.py --fused-only --cases 256:8192:8192,200:8192:8192,512:8192:4096,1024:4096:4096 > gpurun_out/half/ks.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "products or fused or recompute or smoke or c2 or C2" > gpurun_out/half/parity.log 2>&1; tail -2 gpurun_out/half/parity.log

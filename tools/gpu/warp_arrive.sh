mkdir -p gpurun_out/wa
python -c "import __graft_entry__ as g; g.build()"
python tools/k_sweep.py --fused-only --cases 16:8192:8192,64:8192:8192,128:8192:8192,256:8192:8192,512:8192:4096,1024:4096:4096 > gpurun_out/wa/ks.jsonl 2>&1
FS_NVCC_EXTRA="-DFS_PROBE_NO_MMA -DFS_PROBE_NO_COUNT -DFS_PROBE_NO_EXPAND" python -m paper_2104_14667_b200.build --force > /dev/null
python tools/k_sweep.py --fused-only --cases 16:8192:8192,256:8192:8192 > gpurun_out/wa/skeleton.jsonl 2>&1
FS_NVCC_EXTRA="-DFS_PROBE_NO_MMA" python -m paper_2104_14667_b200.build --force > /dev/null
python tools/k_sweep.py --fused-only --cases 16:8192:8192,256:8192:8192 > gpurun_out/wa/nomma.jsonl 2>&1
python -m paper_2104_14667_b200.build --force > /dev/null
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/wa/gpu.log 2>&1; tail -2 gpurun_out/wa/gpu.log

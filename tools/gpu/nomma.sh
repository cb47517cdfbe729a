# timing experiment: fused recompute with and without its main MMAs (results invalid without)
set -e
mkdir -p gpurun_out/nomma
C=16:8192:8192,64:8192:8192,128:8192:8192,256:8192:8192
python tools/k_sweep.py --fused-only --cases $C > gpurun_out/nomma/with.jsonl 2>&1
FS_NVCC_EXTRA=-DFS_PROBE_NO_MMA python -m paper_2104_14667_b200.build --force > /dev/null
python tools/k_sweep.py --fused-only --cases $C > gpurun_out/nomma/without.jsonl 2>&1
FS_NVCC_EXTRA="-DFS_EXP_BATCH=1" python -m paper_2104_14667_b200.build --force > /dev/null
python tools/k_sweep.py --fused-only --cases $C > gpurun_out/nomma/batch1.jsonl 2>&1
python -m paper_2104_14667_b200.build --force > /dev/null

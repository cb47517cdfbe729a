# timing experiment: which part of the fused recompute sets its pace (results invalid
# in the probe builds; the shipped build is restored at the end)
mkdir -p gpurun_out/parts
C=16:8192:8192,128:8192:8192,256:8192:8192
i=0
for d in "" "-DFS_PROBE_NO_MMA" "-DFS_PROBE_NO_MMA -DFS_PROBE_NO_COUNT" "-DFS_PROBE_NO_MMA -DFS_PROBE_NO_EXPAND" \
         "-DFS_PROBE_NO_MMA -DFS_PROBE_NO_EMIT" "-DFS_PROBE_NO_COUNT" "-DFS_PROBE_NO_MMA -DFS_PROBE_NO_COUNT -DFS_PROBE_NO_EXPAND"; do
  FS_NVCC_EXTRA="$d" python -m paper_2104_14667_b200.build --force > /dev/null
  echo "# $d" > gpurun_out/parts/v$i.jsonl
  python tools/k_sweep.py --fused-only --cases $C >> gpurun_out/parts/v$i.jsonl 2>&1
  i=$((i+1))
done
python -m paper_2104_14667_b200.build --force > /dev/null

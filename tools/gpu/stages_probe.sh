# timing experiment: does the 256-panel fused kernel speed up with 4 operand stages?
# (counting dropped so a 2-deep raw ring cannot starve the counters; results invalid)
mkdir -p gpurun_out/st
for d in "-DFS_PROBE_NO_COUNT" "-DFS_PROBE_NO_COUNT -DFS_FUSE_DEPTH_256=2" \
         "-DFS_PROBE_NO_COUNT -DFS_PROBE_NO_MMA -DFS_PROBE_NO_EXPAND -DFS_FUSE_DEPTH_256=2"; do
  FS_NVCC_EXTRA="$d" python -m paper_2104_14667_b200.build --force > /dev/null
  echo "# $d" >> gpurun_out/st/ks.jsonl
  python tools/k_sweep.py --fused-only --cases 256:8192:8192 >> gpurun_out/st/ks.jsonl 2>&1
done
python -m paper_2104_14667_b200.build --force > /dev/null

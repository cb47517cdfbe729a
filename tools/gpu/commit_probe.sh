# timing experiment: cost of tcgen05.commit in the skeleton (results invalid)
mkdir -p gpurun_out/cm
rm -f gpurun_out/cm/ks.jsonl
for d in "-DFS_PROBE_NO_COUNT -DFS_PROBE_NO_MMA -DFS_PROBE_NO_EXPAND -DFS_PROBE_PLAIN_ARRIVE" \
         "-DFS_PROBE_NO_COUNT -DFS_PROBE_NO_MMA -DFS_PROBE_NO_EXPAND -DFS_PROBE_PLAIN_ARRIVE -DFS_PROBE_NO_FENCE"; do
  FS_NVCC_EXTRA="$d" python -m paper_2104_14667_b200.build --force > /dev/null
  echo "# $d" >> gpurun_out/cm/ks.jsonl
  python tools/k_sweep.py --fused-only --cases 16:8192:8192,256:8192:8192 >> gpurun_out/cm/ks.jsonl 2>&1
done
python -m paper_2104_14667_b200.build --force > /dev/null

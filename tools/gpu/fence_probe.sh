# timing experiment: cost of the expanders' proxy fence (results invalid without it)
mkdir -p gpurun_out/fe
rm -f gpurun_out/fe/ks.jsonl
for d in "-DFS_PROBE_NO_COUNT -DFS_PROBE_NO_MMA -DFS_PROBE_NO_EXPAND -DFS_PROBE_NO_FENCE" \
         "-DFS_PROBE_NO_FENCE" "-DFS_PROBE_NO_COUNT -DFS_PROBE_NO_MMA -DFS_PROBE_NO_EXPAND -DFS_EXP_BATCH=1"; do
  FS_NVCC_EXTRA="$d" python -m paper_2104_14667_b200.build --force > /dev/null
  echo "# $d" >> gpurun_out/fe/ks.jsonl
  python tools/k_sweep.py --fused-only --cases 16:8192:8192,256:8192:8192 >> gpurun_out/fe/ks.jsonl 2>&1
done
python -m paper_2104_14667_b200.build --force > /dev/null

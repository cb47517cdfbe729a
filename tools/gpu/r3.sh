set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r3_build.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_gram_tc -s 1 -c 1 -o gpurun_out/r3_gram python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r3_ncu_gram.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_overlap -s 1 -c 1 -o gpurun_out/r3_overlap python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r3_ncu_ov.log 2>&1
ls -la gpurun_out

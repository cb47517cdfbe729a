set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_build.log 2>&1
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
timeout 400 python bench.py --impl reference > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2_ncu_bench.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_gram_tc -s 2 -c 1 -o gpurun_out/r2_gram python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2_ncu_gram.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_overlap -s 2 -c 1 -o gpurun_out/r2_overlap python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/r2_ncu_ov.log 2>&1
ls -la gpurun_out

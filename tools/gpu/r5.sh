set -x
mkdir -p gpurun_out
nvidia-smi -q | head -40 > gpurun_out/r5_smi.txt 2>&1
lscpu > gpurun_out/r5_lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r5_build.log 2>&1
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5_smoke.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r5_pytest.log 2>&1
timeout 600 python bench.py > gpurun_out/r5_bench.json 2> gpurun_out/r5_bench.err
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r5_ref.json 2> gpurun_out/r5_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/r5_ncu_bench.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_gram_tc -s 2 -c 1 -o gpurun_out/r5_gram python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r5_ncu_gram.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_overlap -s 1 -c 1 -o gpurun_out/r5_overlap python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/r5_ncu_ov.log 2>&1
ls -la gpurun_out

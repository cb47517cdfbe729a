# final evidence for the shipped build: default bench (C2), C3 bench, k-sweep, smoke,
# ncu launch list + full capture of the C2 fused recompute
O=gpurun_out/final5
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$? >> $O/smoke.log
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --config c3 --no-cpu > $O/bench_c3.json 2> /dev/null
python bench.py --config c1 > $O/bench_c1.json 2> /dev/null
python tools/k_sweep.py > $O/k_sweep.jsonl 2> /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv \
    python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gram_tc -s 2 -c 1 \
    -o $O/c2_recompute_fused python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ls $O

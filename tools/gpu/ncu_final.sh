# ncu evidence for the shipped build: launch list of the default bench command and one
# full capture of the C2 fused recompute (numbers printed under ncu are not bench values)
O=gpurun_out/ncu_final
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv \
    python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gram_tc -s 2 -c 1 \
    -o $O/c2_recompute_fused python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ls -la $O

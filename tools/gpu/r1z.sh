set -x
O=gpurun_out/r1z
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu > $O/ncu_launch_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu > $O/ncu_launch_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gram_tc -s 2 -c 1 -o $O/c2_recompute_fused python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pack_vec -s 20 -c 1 -o $O/c2_pack_vec python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu > $O/ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_overlap -s 1 -c 1 -o $O/c3_overlap python bench.py --config c3 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gram_pair -s 1 -c 1 -o $O/c3_gram_pair python bench.py --config c3 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu4.log 2>&1
ls -la $O

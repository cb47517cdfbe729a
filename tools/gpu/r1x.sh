set -x
O=gpurun_out/r1x
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pack_engines or products_c1 or products_match_oracle" > $O/pytest.log 2>&1
timeout 600 python tools/sweep_bench.py --engine 0 > $O/sweep_e0.json 2> $O/sweep_e0.err
timeout 600 python tools/sweep_bench.py --engine 2 > $O/sweep_e2.json 2> $O/sweep_e2.err
ls -la $O

# refresh the DESIGN-quoted measurements on the shipped build (subset of tools/reproduce.sh
# without the test suite, ncu and sanitizers, which have their own runs)
O=gpurun_out/refresh
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python bench.py                                   > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --impl reference                  > $O/bench_c2_reference.json 2> $O/ref.err
python bench.py --config c1                       > $O/bench_c1.json 2> /dev/null
python bench.py --config c3 --no-cpu              > $O/bench_c3.json 2> /dev/null
python bench.py --config c4 --steps 3 --warmup 1  > $O/bench_c4.json 2> /dev/null
python tools/sweep_bench.py                       > $O/sweep_c5.json 2> /dev/null
python tools/dual_bench.py                        > $O/dual_buffer_suite.json 2> /dev/null
python tools/k_sweep.py                           > $O/k_sweep.jsonl 2> /dev/null
python tools/service_bench.py                     > $O/service_c2.json 2> /dev/null
python tools/ingest_bench.py                      > $O/ingest.json 2> /dev/null
python tools/compare_with_reference.py            > $O/compare_with_reference.json 2> /dev/null
python tools/run_reference_tests.py               > $O/reference_suite.log 2>&1
ls -la $O

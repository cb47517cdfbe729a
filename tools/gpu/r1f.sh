set -x
O=gpurun_out/r1f
mkdir -p $O
free -g > $O/free.txt 2>&1
nproc >> $O/free.txt
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_banded.py tests/test_reference_port.py -x -q > $O/pytest_new.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k c3_scale > $O/pytest_c3.log 2>&1
timeout 600 python bench.py --config c3 --no-cpu > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --config c4 --steps 3 --warmup 1 > $O/bench_c4.json 2> $O/bench_c4.err
ls -la $O

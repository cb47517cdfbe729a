set -x
O=gpurun_out/r2a
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_c_abi_link.py tests/test_gpu_engine.py -x -q -k "device_similarity or c_program or sharded or ingest or engine" > $O/pytest.log 2>&1
ls -la $O

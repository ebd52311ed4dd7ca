# the committed state once more: bench line (counters matched by source hash), smoke, the bench-contract GPU test
timeout 900 python bench.py > gpurun_out/r3bb_bench.json 2> gpurun_out/r3bb_bench.err; echo "rc=$?" >> gpurun_out/r3bb_bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3bb_smoke.txt 2>&1
timeout 600 python -m pytest tests/test_bench_contract.py tests/test_gpu_segments.py -m gpu -q -p no:cacheprovider > gpurun_out/r3bb_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r3bb_pytest.txt

python -m pytest tests/test_gpu_multidevice.py tests/test_gpu_dropin.py tests/test_gpu_fullsize_golden.py tests/test_gpu_parity.py tests/test_bench_contract.py tests/test_gpu_segments.py -q -m gpu -p no:cacheprovider -rf > gpurun_out/pytest_e.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_e.txt
( time python bench.py --steps 10 --warmup 3 ) > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err

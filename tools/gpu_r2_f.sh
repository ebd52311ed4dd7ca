python -m pytest tests/test_gpu_dropin.py tests/test_gpu_multidevice.py -q -m gpu -p no:cacheprovider -rf -s > gpurun_out/pytest_f.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f.txt

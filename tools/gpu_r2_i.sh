# 8-coil windows with the coils in the MMA M dimension (B) vs before (A); parity of every multi-coil test
python -m pytest tests -q -m gpu -p no:cacheprovider -k "coil or cfg4 or fuzz or parity or fullsize" > gpurun_out/pytest_i.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_i.txt
CONFIGS="4" ROUNDS=3 STEPS=6 bash tools/ab.sh > gpurun_out/i_ab.txt 2>&1
for v in A B; do BLOCH_LIB=$PWD/ab/lib$v.so python tools/shard_probe.py 4 2 4 8 >> gpurun_out/i_ab.txt 2>&1; done

# L2 residency policy for the planes (B, budget via BLOCH_L2_KEEP_MB) vs no cache hints (A)
python -m pytest tests -q -m gpu -p no:cacheprovider -x -k "parity or fuzz or golden" > gpurun_out/pytest_m.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_m.txt
CONFIGS="3 2 1 4" ROUNDS=2 STEPS=6 bash tools/ab.sh > gpurun_out/m_ab.txt 2>&1
for mb in 40 110; do for c in 3 2; do BLOCH_L2_KEEP_MB=$mb BLOCH_LIB=$PWD/ab/libB.so python bench.py --config $c --steps 6 --warmup 3 --no-cpu-baseline --no-per-config --no-projection --e2e-steps 1 --quiet | python -c "import json,sys; d=json.load(sys.stdin); print('cfg$c B keep=${mb}MB kernel_ms %.3f' % d['kernel_ms_per_step'])"; done; done >> gpurun_out/m_ab.txt 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for c in 3 2; do
CMD="python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-per-config --no-projection --e2e-steps 1 --quiet"
BLOCH_LIB=$PWD/ab/libB.so BLOCH_NO_GRAPH=1 $CMD > /dev/null 2>&1 && BLOCH_LIB=$PWD/ab/libB.so BLOCH_NO_GRAPH=1 ncu --metrics $M --clock-control none -k regex:integrate -s 1 -c 1 --csv --log-file gpurun_out/m_cfg${c}_B.csv $CMD > /dev/null 2>&1
done

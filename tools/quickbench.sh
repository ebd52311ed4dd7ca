# quick per-config bench summary (device-resident value, kernel time, roofline frac, e2e)
for c in ${CONFIGS:-1 2 3 4}; do
python bench.py --config $c --steps ${STEPS:-5} --warmup 2 --no-cpu-baseline --quiet | python -c "import json,sys; d=json.load(sys.stdin); print(d['config']['workload'], 'value %.3e' % d['value'], 'kernel_ms %.2f' % d['kernel_ms_per_step'], 'ms/step %.2f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'e2e %.3e' % d['e2e']['value'], 'clk', d['clocks']['sm_mhz'])"
done

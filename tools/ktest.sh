# cfg4 bench at k = 8 / 7 / 6 (walk kernel ms, step ms)
for k in 8 7 6; do
  timeout 300 python bench.py --config 4 --k $k --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('k=$k', 'step %.3f walk %.3f frac %.3f value %.3e' % (d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['value']))"
done

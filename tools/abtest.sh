# A/B: bench each tmpvar/lib*.so in turn (cfg5 walk kernel ms)
for f in tmpvar/lib*.so; do
  cp $f paper_1901_07643_b200/libbnreg.so
  for r in 1 2; do
    timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$f', 'step %.3f walk %.3f frac %.3f' % (d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac']))"
  done
done

for o in none rss both; do
timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --outputs $o 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$o', 'step %.3f walk %.3f' % (d['ms_per_step'], d['roofline']['kernel_ms']))"
done

# A/B of the block-Gram plan (rows per thread) on C1 / C2 / C4: kernel ms and sweeps/s
for c in c2 c4 c1; do
  for e in 0 1 2 4; do
    if [ $e = 0 ]; then unset BAK_BGRAM_E; else export BAK_BGRAM_E=$e; fi
    python bench.py --config $c --variant bgram --steps 3 --warmup 2 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys
try:
    d=json.loads(sys.stdin.read()); print('$c E=$e', d['value'], d['roofline']['kernel_ms'], d['clocks']['sm_mhz'])
except Exception as ex: print('$c E=$e failed')"
  done
done

# GRAM pass kernel alone (bench roofline kernel_ms) for alternative builds
set -u
for v in "$@"; do
  for c in c3 c3f32; do
    echo -n "$v $c: "
    BAK_LIB_PATH=$PWD/tools/ab/$v.so timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e --no-exact 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['roofline']['kernel_ms'], d['roofline']['achieved'], d['value'], d['step_ms'])"
  done
done

# A/B of library builds on the c3s8 bench (kernel ms of the exact sweep): ab_c3s8.sh v1 v2 ...
for v in "$@"; do
  if [ "$v" = base ]; then unset BAK_LIB_PATH; else export BAK_LIB_PATH=$PWD/paper_2104_12570_b200/libbak200_$v.so; fi
  python bench.py --config c3s8 --steps 3 --warmup 2 --no-e2e --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
done

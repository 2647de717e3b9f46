# A/B: time the latency-bound sweep shapes with alternative builds of libbak200.so
set -u
for v in "$@"; do
  for args in "--obs 1000 --vars 20000 --sweeps 2 --variant cta" "--obs 4096 --vars 4096 --sweeps 2 --variant cluster" "--obs 10000 --vars 100 --sweeps 50 --variant cluster"; do
    echo -n "$v $args: "
    BAK_LIB_PATH=$PWD/tools/ab/$v.so timeout 120 python tools/sweep_probe.py $args 2>&1 | tail -1
  done
done

# Round profiles: launch list of the default bench, full ncu sections of the
# top kernels.  Each profiled command has already exited 0 without ncu.
# Outputs under gpurun_out/prof/.
set -u
mkdir -p gpurun_out/prof
O=gpurun_out/prof
NCU="ncu --clock-control none"
# 1. launch list of the default bench (C3 fp64), one timed step
timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -c 400 --csv \
  --log-file $O/launches_c3.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-exact > $O/launches_c3.out 2>&1
echo "launches rc=$?"
# 2. full sections: GRAM pass + DMMA G kernel (C3 shape)
timeout 900 $NCU --set full --import-source on -k regex:"gram_pass_tma|gram_dmma" -c 2 -o $O/c3_gram_full \
  python tools/sweep_probe.py --obs 16777216 --vars 256 --sweeps 2 --variant gram > $O/c3_gram_full.out 2>&1
echo "gram full rc=$?"
# 3. full sections: blocked on-chip kernel (p1 shape) and the scoring kernels
timeout 600 $NCU --set full --import-source on -k regex:"block_kernel" -c 1 -o $O/p1_block_full \
  python tools/bakp_phases.py 10000 1000 50 f32 > $O/p1_block_full.out 2>&1
echo "block full rc=$?"
timeout 600 $NCU --set full --import-source on -k regex:"score_" -c 3 -o $O/score_full \
  python tools/score_probe.py > $O/score_full.out 2>&1
echo "score full rc=$?"

# DRAM bytes per launch for the on-chip-e kernels (north star: "ncu must show
# (ncu cannot replay cooperative launches with clusters: under ncu the library uses the one-level exchange
#  automatically (coop_clusters_ok), whose DRAM traffic is the same; the FLAT variables below are explicit)
# ... that e traffic stays on-chip").  Each command first runs without ncu.
set -u
mkdir -p gpurun_out/prof
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
python tools/batched_time.py 65536 20 > /dev/null && \
ncu --clock-control none --metrics $M -k regex:batched_kernel --csv python tools/batched_time.py 65536 20 \
  > gpurun_out/prof/dram_c5.csv 2>/dev/null; echo "c5 rc=$?"
python tools/sweep_probe.py --obs 262144 --vars 128 --sweeps 4 --dtype f64 --variant grid --reps 1 > /dev/null && \
BAK_GRID_FLAT=1 ncu --clock-control none --metrics $M -k regex:sweep_kernel --csv python tools/sweep_probe.py --obs 262144 --vars 128 \
  --sweeps 4 --dtype f64 --variant grid --reps 1 > gpurun_out/prof/dram_grid.csv 2>/dev/null; echo "grid rc=$?"
python tools/sweep_probe.py --obs 10000 --vars 100 --sweeps 100 --dtype f64 --reps 1 > /dev/null && \
ncu --clock-control none --metrics $M -k regex:sweep_kernel --csv python tools/sweep_probe.py --obs 10000 --vars 100 \
  --sweeps 100 --dtype f64 --reps 1 > gpurun_out/prof/dram_c1.csv 2>/dev/null; echo "c1 rc=$?"
python tools/sweep_probe.py --obs 4194304 --vars 32 --sweeps 2 --dtype f64 --variant stream --reps 1 > /dev/null && \
BAK_STREAM_FLAT=1 ncu --clock-control none --metrics $M -k regex:stream_kernel --csv python tools/sweep_probe.py --obs 4194304 \
  --vars 32 --sweeps 2 --dtype f64 --variant stream --reps 1 > gpurun_out/prof/dram_stream.csv 2>/dev/null; echo "stream rc=$?"

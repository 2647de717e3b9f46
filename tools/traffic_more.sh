# DRAM bytes per launch of the dominant kernel for the other bench configs
# (roofline.traffic): c3f32 / p3 GRAM pass, c5 batched kernel (200 sweeps)
set -u
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
mkdir -p gpurun_out/prof
python tools/sweep_probe.py --obs 16777216 --vars 256 --sweeps 2 --reps 1 --variant gram --dtype f32 > /dev/null 2>&1 && \
ncu --clock-control none --metrics $M -k regex:gram_pass_tma -c 2 --csv python tools/sweep_probe.py --obs 16777216 --vars 256 \
  --sweeps 2 --reps 1 --variant gram --dtype f32 > gpurun_out/prof/traffic_c3f32.csv 2>/dev/null; echo c3f32=$?
python tools/batched_time.py 65536 200 > /dev/null 2>&1 && \
ncu --clock-control none --metrics $M -k regex:batched_kernel -c 1 --csv python tools/batched_time.py 65536 200 \
  > gpurun_out/prof/traffic_c5.csv 2>/dev/null; echo c5=$?

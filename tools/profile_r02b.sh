# Round-2 (second half) ncu captures; every profiled command first exits 0 without ncu.
#   launch lists:  default bench (c3 fp64), c3s8 (XT exact sweep), c4 block-Gram
#   full sections: the XT sweep kernel, bgram_kernel
set -x
mkdir -p gpurun_out
B="--steps 1 --warmup 3 --no-e2e --no-cpu --no-exact"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
python bench.py $B > gpurun_out/p_c3.log 2>&1 && \
ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_c3.csv python bench.py $B > gpurun_out/n0.log 2>&1
python bench.py --config c3s8 $B > gpurun_out/p_c3s8.log 2>&1 && \
ncu --metrics $M --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_c3s8.csv python bench.py --config c3s8 $B > gpurun_out/n2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o gpurun_out/r02_prof_xt \
    python bench.py --config c3s8 $B > gpurun_out/n4.log 2>&1
python bench.py --config c4 --variant bgram $B > gpurun_out/p_c4bg.log 2>&1 && \
ncu --metrics $M --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_c4_bgram.csv python bench.py --config c4 --variant bgram $B > gpurun_out/n6.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:bgram_kernel -c 1 -o gpurun_out/r02_prof_bgram \
    python bench.py --config c4 --variant bgram $B > gpurun_out/n5.log 2>&1
echo profile_r02b done

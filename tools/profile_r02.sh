# Round-2 ncu captures (one gpurun call; every profiled command first exits 0 without ncu).
#   launch lists:  c3f32 (tcgen05 G + passes), c3s8 (XS exact sweep), c4 bgram
#   full sections: gram_tc_kernel, the XS sweep kernel, bgram_kernel
set -x
mkdir -p gpurun_out
B="--steps 1 --warmup 3 --no-e2e --no-cpu --no-exact"
python bench.py --config c3f32 $B > gpurun_out/p_c3f32.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/r02_launches_c3f32.csv python bench.py --config c3f32 $B > gpurun_out/n1.log 2>&1
python bench.py --config c3s8 $B > gpurun_out/p_c3s8.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/r02_launches_c3s8.csv python bench.py --config c3s8 $B > gpurun_out/n2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gram_tc_kernel -c 1 -o gpurun_out/r02_prof_tc \
    python bench.py --config c3f32 $B > gpurun_out/n3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o gpurun_out/r02_prof_xs \
    python bench.py --config c3s8 $B > gpurun_out/n4.log 2>&1
python bench.py --config c4 --variant bgram $B > gpurun_out/p_c4bg.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:bgram_kernel -c 1 -o gpurun_out/r02_prof_bgram \
    python bench.py --config c4 --variant bgram $B > gpurun_out/n5.log 2>&1
echo profile_r02 done

# libbak200_phases$PHNAME.so: the library with -DBAK_PHASES in the sweep kernels (per-phase
# clock64 counters, tools/phases.py).  BAK_LIB_PATH=paper_2104_12570_b200/libbak200_phases$PHNAME.so
set -e
cd "$(dirname "$0")/.."
python -m paper_2104_12570_b200.build > /dev/null
B=paper_2104_12570_b200/_build
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include -DBAK_PHASES"
nvcc $F $PHDEFS -c paper_2104_12570_b200/csrc/bak_sweep.cu -o /tmp/bak_sweep_ph.o &
nvcc $F -c paper_2104_12570_b200/csrc/bak_bgram.cu -o /tmp/bak_bgram_ph.o &
wait
OBJS=$(ls $B/*.o | grep -v "bak_sweep.o\|bak_bgram.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2104_12570_b200/libbak200_phases$PHNAME.so $OBJS /tmp/bak_sweep_ph.o /tmp/bak_bgram_ph.o -lpthread
echo built paper_2104_12570_b200/libbak200_phases$PHNAME.so

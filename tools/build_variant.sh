# build_variant.sh NAME "-DFLAG=.. ..." [file.cu ...]: libbak200_NAME.so with extra defines in the
# listed sources (default bak_sweep.cu); other objects come from the regular build.  A/B runs:
# BAK_LIB_PATH=$PWD/paper_2104_12570_b200/libbak200_NAME.so
set -e
cd "$(dirname "$0")/.."
NAME=$1; DEFS=$2; shift 2
SRCS=${@:-bak_sweep.cu}
B=paper_2104_12570_b200/_build
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include $DEFS"
EXCL=""; NEW=""
for s in $SRCS; do
  o=/tmp/${NAME}_${s%.cu}.o
  nvcc $F -c paper_2104_12570_b200/csrc/$s -o $o &
  EXCL="$EXCL\|${s%.cu}.o"; NEW="$NEW $o"
done
wait
OBJS=$(ls $B/*.o | grep -v "XXXX$EXCL")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2104_12570_b200/libbak200_$NAME.so $OBJS $NEW -lpthread
echo built paper_2104_12570_b200/libbak200_$NAME.so

# C5 batched: cap on resident systems per SM (x working set vs the 126 MB L2)
set -u
for n in auto 0 11 12 13 14 auto; do
  echo -n "per_sm=$n: "
  if [ $n = auto ]; then timeout 300 python tools/batched_time.py 2>&1 | tail -1
  else BAK_BATCH_PER_SM=$n timeout 300 python tools/batched_time.py 2>&1 | tail -1; fi
done

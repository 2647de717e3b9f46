for n in 262144 1048576 2097152; do
  for envs in "X=0" "BAK_GRID_FLAT=1" "BAK_GRID_FLAT=1 BAK_GRID_AG=1"; do
    for prec in f64 f32; do
      r=$(env $envs timeout 120 python tools/grid_compare.py --one $n $prec grid 2>&1 | tail -1)
      echo "$envs $r"
    done
  done
done

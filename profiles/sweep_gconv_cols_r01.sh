# FFMA gconv plans for the paper's four gconv columns (tile_sizes = [rows per block, rf, rw])
for op in gconv14 gconv7 gconv56 gconv28; do
  echo "== $op"
  timeout 200 python profiles/sweep.py $op '[{"tile_sizes":[7,4,7]},{"tile_sizes":[2,1,1]},{"tile_sizes":[4,1,1]},{"tile_sizes":[7,2,7]},{"tile_sizes":[2,8,7]},{"tile_sizes":[4,4,4]},{"tile_sizes":[8,4,4]},{"tile_sizes":[2,4,7]},{"tile_sizes":[14,2,7]},{"tile_sizes":[1,8,4]}]'
done

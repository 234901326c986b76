for v in exp3 exp2; do for c in "24 1 20001" "44 4 20001" "20 2 20001"; do
  echo "== $v $c"; RAFI_LIB_PATH=$PWD/paper_2605_30294_b200/_variants/librafi_$v.so python scripts/chunk_dbg.py $c 2>&1 | tail -1
done; done

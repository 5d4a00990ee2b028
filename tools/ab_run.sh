for rep in 1 2; do
 for v in cur ilp3c1 ilp4c1; do
  echo -n "$v "; BD_LIB_PATH=build_variants/lib_$v.so python tools/profile_am.py --scenes 64 --lanes 8 --cycles 2 2>&1 | tail -1
 done
done

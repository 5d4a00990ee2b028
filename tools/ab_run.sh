for rep in 1 2; do
 for v in cur itms; do
  BD_LIB_PATH=build_variants/lib_$v.so python tools/profile_am.py --scenes 1 --batch 1000 --cycles 20 2>&1 | tail -1
  BD_LIB_PATH=build_variants/lib_$v.so python tools/profile_am.py --scenes 64 --cycles 2 2>&1 | tail -1
  BD_LIB_PATH=build_variants/lib_$v.so python tools/profile_am.py --scenes 1 --batch 10000 --obs 50 --cycles 3 2>&1 | tail -1
 done
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_persistent.py tests/test_gpu_fleet.py tests/test_gpu_random_parity.py -q -p no:cacheprovider 2>&1 | tail -2
python tools/probes/persist_time.py 60

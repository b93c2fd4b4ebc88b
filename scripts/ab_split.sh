timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_native_loop.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "time_split or row_plan or native or device_loop or transient_golden or c3 or closed_loop" 2>&1 | tail -2
for L in new=paper_2510_08288_b200/_lib/librefgov_b200.so old=paper_2510_08288_b200/_lib/variants/dl2/librefgov_b200.so; do
  echo "== ${L%%=*}"; RG_LIB_PATH=${L#*=} timeout 200 python scripts/ab_split.py
  RG_LIB_PATH=${L#*=} timeout 300 python scripts/device_loop_diag.py 2>&1 | grep "device_loop=1" | cut -c1-120
done

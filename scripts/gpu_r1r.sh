AB_TEST="tests/test_gpu_forward.py" bash scripts/gpu_ab.sh sort2 "base=" "items15=-DSK_SORT_SMALL_N=0" "items5=-DSK_SORT_SMALL_ITEMS=5" > gpurun_out/ab_sort2.txt 2>&1; cat gpurun_out/ab_sort2.txt

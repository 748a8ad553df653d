export AB_TEST="tests/test_gpu_forward.py tests/test_gpu_backward.py"
bash scripts/gpu_ab.sh ws "base=" "fwdws=-DSK_FWD_WARP_STAGED=1" "bwdws=-DSK_BWD_WARP_STAGED=1" "fwdws4=-DSK_FWD_WARP_STAGED=1 -DSK_FWD_PIX16=4" "bothws=-DSK_FWD_WARP_STAGED=1 -DSK_BWD_WARP_STAGED=1" > gpurun_out/ab_ws.txt 2>&1
cat gpurun_out/ab_ws.txt
SK_TRACE_EVENTS=1 timeout 600 python bench.py --workload event --no-cpu-baseline --steps 2 > gpurun_out/event_trace.json 2> gpurun_out/event_trace.err
grep "\[event\]" gpurun_out/event_trace.err | tail -24

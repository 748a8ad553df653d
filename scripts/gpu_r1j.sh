AB_TEST="tests/test_gpu_backward.py" bash scripts/gpu_ab.sh pix "base=" "bpix2=-DSK_BWD_PIX16=2" "bpix2m12=-DSK_BWD_PIX16=2 -DSK_BWD_MINB=6" > gpurun_out/ab_pix.txt 2>&1; cat gpurun_out/ab_pix.txt
timeout 600 python bench.py > gpurun_out/bench_r1j.json 2> gpurun_out/bench_r1j.err; tail -c 300 gpurun_out/bench_r1j.err
python -c "import json; d=json.load(open('gpurun_out/bench_r1j.json')); print(d['value'], d['e2e'], d['phase_ms'])"

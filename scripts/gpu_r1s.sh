timeout 900 python -m pytest tests/test_golden.py tests/test_gpu_forward.py -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
git stash list > /dev/null 2>&1
AB_TEST="" bash scripts/gpu_ab.sh ad "base=" > gpurun_out/ab_ad.txt 2>&1; cat gpurun_out/ab_ad.txt

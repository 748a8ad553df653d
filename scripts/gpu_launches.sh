WARM=150
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -s $((19 * WARM)) -c 60 \
  --log-file gpurun_out/launches_r1f.csv python bench.py --profile --steps 2 --warmup $WARM > /dev/null 2>&1
wc -l gpurun_out/launches_r1f.csv

for v in 1 0; do
  SK_NVCC_EXTRA="-DSK_SCORE_TWO_STREAMS=$v" python -c "import paper_2511_04283_b200 as sk; sk.build(force=True)" > /dev/null
  SK_TRACE_EVENTS=1 timeout 900 python bench.py --workload event --n 8000000 --views 10 --steps 5 --no-cpu-baseline > gpurun_out/event_8m_$v.json 2> gpurun_out/event_8m_$v.err
  echo "two_streams=$v"; grep "score pass" gpurun_out/event_8m_$v.err | awk '{print $(NF-1)}' | tr '\n' ' '; echo
done
python -c "import paper_2511_04283_b200 as sk; sk.build(force=True)" > /dev/null

for m in ce sm; do
SCOUT_RECALL_PROF=1 timeout 900 python bench.py --no-extras --no-cpu-baseline --recall-mode $m > gpurun_out/g8_$m.json 2> gpurun_out/g8_$m.err; echo rc=$?; tail -6 gpurun_out/g8_$m.err
done
SCOUT_RECALL_PROF=1 timeout 900 python bench.py --no-extras --no-cpu-baseline --recall-policy stagger > gpurun_out/g8_st.json 2> gpurun_out/g8_st.err; echo rc=$?; tail -6 gpurun_out/g8_st.err

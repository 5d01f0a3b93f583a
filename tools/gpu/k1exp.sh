# K1 experiment: parity, static + tier bench, K1 launch time and one full capture
T=${1:-k1x}
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_engine.py tests/test_gpu_engine_tier.py -x -q 2>&1 | tail -2
for c in "--tier static" ""; do
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'].get('workload'), d.get('tier') is not None, 'step', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), 'k2', round(d['roofline']['avg_launch_us'],1))"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -k "regex:score_topk|sparse_decode" -c 20 --csv --log-file gpurun_out/launches_$T.csv python bench.py --profile --steps 2 --warmup 1 --tier static > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/launches_$T.csv')) if len(r)>10]
h=rows[0]; ik=h.index('Kernel Name'); iv=h.index('Metric Value')
from collections import defaultdict
d=defaultdict(list)
for r in rows[1:]: d[r[ik][:60]].append(float(r[iv].replace(',','')))
for k,v in d.items(): print(k, len(v), sum(v)/len(v))
PY
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:score_topk -c 1 -f -o gpurun_out/prof_k1_$T python bench.py --profile --steps 2 --warmup 1 --tier static > /dev/null 2>&1
echo done

# CPU co-attention worker on the GPU box: ISA, parity tests, bench line
grep -m1 "model name" /proc/cpuinfo; nproc
grep -m1 flags /proc/cpuinfo | tr ' ' '\n' | grep -E "amx|avx512_bf16" | tr '\n' ' '; echo
timeout 600 python -m pytest tests/test_cpu_coattn.py -q 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/cpuw_bench.json 2> gpurun_out/cpuw_bench.err
tail -1 gpurun_out/cpuw_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'], json.dumps(d.get('cpu_coattention')))"

timeout 900 python bench.py > gpurun_out/g4_bench.json 2> gpurun_out/g4_bench.err; echo rc=$?; tail -12 gpurun_out/g4_bench.err

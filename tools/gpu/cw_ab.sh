# A/B of CPU co-attention worker builds: per-unit cost and the composed step
# usage: bash tools/gpu/cw_ab.sh <variant>...   (paper_2603_27138_b200/_ab/libscout_b200_<variant>.so)
for v in "$@"; do
  L=paper_2603_27138_b200/_ab/libscout_b200_$v.so
  echo "== $v"
  SCOUT_B200_LIB=$L timeout 300 python tools/debug/cpu_unit_cost.py 2>&1 | grep threads
  SCOUT_B200_LIB=$L timeout 400 python tools/debug/cw_ab.py 2>&1 | grep composed
done

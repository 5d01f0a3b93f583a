cd $GRAFT_REPO_ROOT
for v in base s6d4 s8d4 s5; do
  if [ $v = base ]; then L=paper_2603_27138_b200/libscout_b200.so; else L=paper_2603_27138_b200/_ab/libscout_b200_$v.so; fi
  echo "== $v"; SCOUT_B200_LIB=$L timeout 400 python tools/debug/layerwise_ctas.py 80 96 104 112 120 80 2>&1 | grep -v Warn | tail -7
done

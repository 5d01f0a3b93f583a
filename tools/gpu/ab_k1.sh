# A/B of K1 alone (tools/debug/time_k1.py): built library vs libscout_b200_old.so
L=paper_2603_27138_b200
cp $L/libscout_b200.so /tmp/new.so
for r in 1 2 3; do
  cp /tmp/new.so $L/libscout_b200.so; echo "new: $(timeout 120 python tools/debug/time_k1.py 2>&1 | grep batch)"
  cp $L/libscout_b200_old.so $L/libscout_b200.so; echo "old: $(timeout 120 python tools/debug/time_k1.py 2>&1 | grep batch)"
done
cp /tmp/new.so $L/libscout_b200.so

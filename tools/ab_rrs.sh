# alternating A/B of lib/old.so vs the current lib for implicit-store RRS solves
L=paper_2111_11728_b200/lib
cp $L/libfetigpu.so /tmp/new.so
for r in 1 2; do
  cp $L/old.so $L/libfetigpu.so; echo OLD; python tools/rrs_hash.py
  cp /tmp/new.so $L/libfetigpu.so; echo NEW; python tools/rrs_hash.py
done

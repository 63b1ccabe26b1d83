# A/B of lib/old.so against the current lib/libfetigpu.so for the K5 block
# apply on C4: time at k = 2048 and a bit-identity hash of Q at k = 64.
L=paper_2111_11728_b200/lib
cp $L/libfetigpu.so /tmp/new.so
cp $L/old.so $L/libfetigpu.so
echo OLD; python tools/prof_block_c4.py --k 64 --hash; python tools/prof_block_c4.py; python tools/prof_block_c4.py
cp /tmp/new.so $L/libfetigpu.so
echo NEW; python tools/prof_block_c4.py --k 64 --hash; python tools/prof_block_c4.py; python tools/prof_block_c4.py

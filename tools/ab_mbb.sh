L=paper_2111_11728_b200/lib
cp $L/libfetigpu.so /tmp/new.so
cp $L/old.so $L/libfetigpu.so
echo OLD; python tools/mbb_variant.py
cp /tmp/new.so $L/libfetigpu.so
echo NEW; python tools/mbb_variant.py

# A/B of lib/old.so (baseline) against the current lib/libfetigpu.so on one box:
# operator hashes (bit-identity), C4 build timing, k_nd_small launch list.
L=paper_2111_11728_b200/lib
cp $L/libfetigpu.so /tmp/new.so
cp $L/old.so $L/libfetigpu.so
python tools/apply_hash.py > gpurun_out/hash_old.txt 2>&1
python tools/prof_build.py --reps 4 > gpurun_out/build_old.txt 2>&1
cp /tmp/new.so $L/libfetigpu.so
python tools/apply_hash.py > gpurun_out/hash_new.txt 2>&1
python tools/prof_build.py --reps 4 > gpurun_out/build_new.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:${NCU_K:-k_nd_small} -c ${NCU_C:-8} --csv python tools/prof_build.py > gpurun_out/ab_launches.csv 2>&1

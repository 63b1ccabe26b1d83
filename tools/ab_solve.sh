L=paper_2111_11728_b200/lib
cp $L/libfetigpu.so /tmp/new.so
cp $L/old.so $L/libfetigpu.so
python tools/solve_hash.py > gpurun_out/sh_old.txt 2>&1
FETIGPU_HOST_LOOP=1 python tools/solve_hash.py > gpurun_out/sh_old_host.txt 2>&1
cp /tmp/new.so $L/libfetigpu.so
python tools/solve_hash.py > gpurun_out/sh_new.txt 2>&1
FETIGPU_HOST_LOOP=1 python tools/solve_hash.py > gpurun_out/sh_new_host.txt 2>&1
python tools/solve_hash.py > gpurun_out/sh_new2.txt 2>&1

# A/B of one env switch on the same build: operator hashes and C4 build timing
# with and without $AB_ENV (e.g. AB_ENV=FETIGPU_BPC_TILE=1).
python tools/apply_hash.py > gpurun_out/hash_new.txt 2>&1
env $AB_ENV python tools/apply_hash.py > gpurun_out/hash_old.txt 2>&1
for i in 1 2; do
  python tools/prof_build.py --reps 3 >> gpurun_out/build_new.txt 2>&1
  env $AB_ENV python tools/prof_build.py --reps 3 >> gpurun_out/build_old.txt 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:${NCU_K:-k_bpc_update} --csv python tools/prof_build.py > gpurun_out/ab_new.csv 2>&1
env $AB_ENV ncu --metrics gpu__time_duration.sum --clock-control none -k regex:${NCU_K:-k_bpc_update} --csv python tools/prof_build.py > gpurun_out/ab_old.csv 2>&1

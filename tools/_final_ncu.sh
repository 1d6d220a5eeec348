# ncu --set full captures (split from _final.sh: gpurun returns <= 64 MiB per call);
# WITH_C3=1: only the 3-D tensor-engine capture
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/prof_c2_states.ncu-rep gpurun_out/prof_c2_flux.ncu-rep gpurun_out/prof_c2_update.ncu-rep gpurun_out/prof_c3_states_128.ncu-rep
[ "${WITH_C3:-0}" = 1 ] || timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stage_row -s 3 -c 1 -o gpurun_out/prof_c2_states python tools/profile_step.py --config 2 --steps 2 > gpurun_out/ncu1.log 2>&1
[ "${WITH_C3:-0}" = 1 ] || timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_flux -s 3 -c 1 -o gpurun_out/prof_c2_flux python tools/profile_step.py --config 2 --steps 2 > gpurun_out/ncu2.log 2>&1
[ "${WITH_C3:-0}" = 1 ] || timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update -s 3 -c 1 -o gpurun_out/prof_c2_update python tools/profile_step.py --config 2 --steps 2 > gpurun_out/ncu4.log 2>&1
[ "${WITH_C3:-0}" = 1 ] && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_states_u -s 3 -c 1 -o gpurun_out/prof_c3_states_128 python tools/profile_step.py --config 3 --n 128 --steps 2 > gpurun_out/ncu3.log 2>&1
ls gpurun_out/*.ncu-rep

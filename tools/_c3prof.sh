cd $GRAFT_REPO_ROOT
rm -f gpurun_out/prof_c3_states_128.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_states_u -s 3 -c 1 -o gpurun_out/prof_c3_states_128 python tools/profile_step.py --config 3 --n 128 --steps 2 > gpurun_out/ncu3.log 2>&1; tail -2 gpurun_out/ncu3.log
make -B EXTRA=-DKFVM_PHASE_TIMING -j8 > gpurun_out/make_phase.log 2>&1 || tail gpurun_out/make_phase.log
python tools/phase_times.py 3 128 2
python tools/phase_times.py 5 128 2

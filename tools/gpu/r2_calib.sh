# ncu pipe metrics on the DMMA/DFMA interleave ubench (calibration of
# sm__pipe_tensor/fp64_cycles_active against the measured datapath rate)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ubench/dmma_dfma_ratio.cu -o /tmp/ratio
timeout 120 /tmp/ratio > gpurun_out/ratio_plain.txt 2>&1
timeout 600 ncu --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum --csv /tmp/ratio > gpurun_out/ratio_ncu.csv 2>&1
cat gpurun_out/ratio_plain.txt

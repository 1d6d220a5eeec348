# SPEC acceptance measurements on the GPU path -> gpurun_out/acceptance.json
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python tools/acceptance.py ${CHECKS} > gpurun_out/acceptance.json 2> gpurun_out/acceptance.log; echo "rc=$?" >> gpurun_out/acceptance.log
cat gpurun_out/acceptance.log

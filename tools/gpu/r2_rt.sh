cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/rt.txt; : > $out
for o in "ring_tiles=1" "ring_tiles=8" "ring_tiles=16" "ring_tiles=32" "ring_tiles=64"; do
  echo "-- $o" >> $out
  timeout 300 python tools/time_step.py --config 4 --steps 3 --opt $o >> $out 2>&1
done
cat $out

# device time per step of the config 4 recipe (3-D R=2 outflow Voronoi) over grid sizes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/sizes.txt; : > $out
for n in 64 96 128 200 256 384 512; do
  echo "-- n=$n" >> $out
  timeout 300 python tools/time_step.py --config 4 --n $n --steps 3 >> $out 2>&1
done
for n in 64 128 256; do
  echo "-- R=3 periodic n=$n" >> $out
  timeout 300 python tools/time_step.py --config 5 --n $n --steps 2 >> $out 2>&1
done
cat $out

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/kz2d.txt; : > $out
for kz in 4 5 6 7 8 10 12 16; do
  echo "-- kz=$kz" >> $out
  timeout 300 python tools/time_step.py --config 2 --steps 100 --opt kz=$kz >> $out 2>&1
done
cat $out

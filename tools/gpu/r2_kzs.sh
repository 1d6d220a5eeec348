cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/kzs.txt; : > $out
for kz in 8 12 16 24 32; do
  echo "-- c3 n=256 kz=$kz" >> $out
  timeout 300 python tools/time_step.py --config 3 --steps 5 --opt kz=$kz >> $out 2>&1
done
for kz in 16 24 32 48; do
  echo "-- c4 n=384 kz=$kz" >> $out
  timeout 300 python tools/time_step.py --config 4 --n 384 --steps 3 --opt kz=$kz >> $out 2>&1
done
for kz in 8 16 32; do
  echo "-- c5 n=128 kz=$kz" >> $out
  timeout 300 python tools/time_step.py --config 5 --n 128 --steps 3 --opt kz=$kz >> $out 2>&1
done
cat $out

# R=3 regression bisection: config 5 recipe at 256^3 with older trees' libraries
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
out=gpurun_out/bisect.txt; : > $out
for t in wt_eb5cecd wt_957ef98 wt_fc72f82 wt_ae053f1; do
  echo "== $t" >> $out
  (cd build/trees/$t && timeout 300 python tools/time_step.py --config 5 --n 256 --steps 2) >> $out 2>&1
done
echo "== HEAD" >> $out
timeout 300 python tools/time_step.py --config 5 --n 256 --steps 2 >> $out 2>&1
cat $out

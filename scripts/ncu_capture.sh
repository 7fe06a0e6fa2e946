# ncu evidence for one bench workload ($WL, default c2): the launch list of the
# bench command (cold, serialised) and one --set full capture of the level-0
# launch of each stage's kernel (sweep_l0, sgm_l0), named by stage so
# scripts/ncu_summary.py keys them the way bench.py reads them.
#   WL=c3 bash scripts/ncu_capture.sh   -> gpurun_out/ncu_$WL/
WL=${WL:-c2}
OUT=gpurun_out/ncu_$WL
mkdir -p $OUT
B="python bench.py --workload $WL --steps 2 --warmup 1 --inflight 1 --ring 2 --no-cpu-baseline"
case $WL in
  c2|c2pg|c5) SW=sweep_census_tiled; SKIP=5 ;;   # 3 tiled sweeps / SGM launches per bundle: L2, L1, L0
  c2ncc|c4)   SW=sweep_ncc_tiled; SKIP=5 ;;
  c3)         SW=sweep_ncc_tiled; SKIP=2 ;;      # one level
  c1)         SW=sweep_census_tiled; SKIP=2 ;;
esac
SG=sgm_line_kernel

timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches.csv $B > $OUT/ncu_launch.log 2>&1; echo launches rc=$?
for st in sweep_l0:$SW sgm_l0:$SG; do
  name=${st%%:*}; k=${st#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k \
    --launch-skip $SKIP -c 1 -f -o $OUT/full_$name $B > $OUT/ncu_full_$name.log 2>&1
  echo "full $name ($k) rc=$?"
done

# BASELINE config 4 on one B200 through the CLI: a Mip-NeRF-360-sized synthetic
# scene (3M GT Gaussians, 200 views 1297x840, every 8th view held out), then a
# full 30K-iteration training run with the default schedule (densify / prune
# events every 500 iterations until 15K, late prunes every 3K).
set -e
CLI=paper_2511_04283_b200/splatkit_b200
OUT=gpurun_out/config4
rm -rf $OUT; mkdir -p $OUT
SM=$(python -c "print((500/3e6)**(1/3))")
FOCAL=$(python -c "print(1.1*840*2.6)")
T0=$(date +%s.%N); $CLI synth --out $OUT/data --gaussians 3000000 --views 200 --width 1297 --height 840 \
  --scale-mult $SM --focal $FOCAL --seed 1 > $OUT/synth.log 2>&1; T1=$(date +%s.%N)
cat > $OUT/train.cfg <<'CFG'
seed = 17
CFG
$CLI train --data $OUT/data --out $OUT/run --config $OUT/train.cfg > $OUT/train.log 2>&1; T2=$(date +%s.%N)
echo "synth_s $(python -c "print($T1-$T0)") train_cli_s $(python -c "print($T2-$T1)")" | tee $OUT/wall.txt
cat $OUT/run/metrics.json | head -8
cat $OUT/run/timing.json
tail -3 $OUT/run/log.csv
rm -rf $OUT/data/images $OUT/run/renders $OUT/data/*.ply $OUT/run/checkpoint.ply

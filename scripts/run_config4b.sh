# Config-4 training with the screen-size prune disabled (diagnostic for the
# default run's Gaussian-count collapse).
set -e
CLI=paper_2511_04283_b200/splatkit_b200
OUT=gpurun_out/config4b
rm -rf $OUT; mkdir -p $OUT
SM=$(python -c "print((500/3e6)**(1/3))")
FOCAL=$(python -c "print(1.1*840*2.6)")
$CLI synth --out $OUT/data --gaussians 3000000 --views 200 --width 1297 --height 840 \
  --scale-mult $SM --focal $FOCAL --seed 1 > $OUT/synth.log 2>&1
printf "seed = 17\nprune_screen_size = 1000000\n" > $OUT/nosize.cfg
$CLI train --data $OUT/data --out $OUT/nosize --config $OUT/nosize.cfg > $OUT/nosize.log 2>&1
printf "seed = 17\nvcp = false\n" > $OUT/novcp.cfg
$CLI train --data $OUT/data --out $OUT/novcp --config $OUT/novcp.cfg > $OUT/novcp.log 2>&1
for r in nosize novcp; do echo $r; awk -F, 'NR%3000==2' $OUT/$r/log.csv; grep mean_psnr $OUT/$r/metrics.json; done
rm -rf $OUT/data $OUT/*/renders $OUT/*/checkpoint.ply

# ncu --set full of the mixed-slot kernel on the probe shapes (4th launch = first timed)
N=4194304
for o in shuffled grouped; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:predict_mixed -s 3 -c 1 \
    -o gpurun_out/mixed_${o}29 python tools/mixed_probe.py $N 200 29 $o > gpurun_out/mixed_ncu_${o}29.log 2>&1
done

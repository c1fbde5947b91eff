N=4194304
for F in 200 256; do for st in 3 4 5 6; do GNB_PRED_MIXED=2 GNB_MIXED_STAGES=$st python tools/mixed_probe.py $N $F 1 grouped; done; done
for S in 2 8 29; do for o in grouped shuffled; do python tools/mixed_probe.py $N 200 $S $o; GNB_PRED_MIXED=0 python tools/mixed_probe.py $N 200 $S $o; done; done
for S in 2 8; do for st in 3 4 5 6; do GNB_MIXED_STAGES=$st python tools/mixed_probe.py $N 200 $S shuffled; done; done

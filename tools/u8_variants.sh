# uint8 / uint16 K-PRED (cfg4 shape, 16M rows) under the CP=2 geometry variants
# (GNB_PRED_VARIANT: 0 = R1 NW4 S2 default, 2 = R2 NW2 S2, 3 = R2 NW4 S2), exact + fma
for v in 0 2 3; do
  for m in "" "--fma"; do
    for d in "" "--u16"; do
      echo "variant $v $m $d: $(GNB_PRED_VARIANT=$v timeout 300 python tools/u8_probe.py $m $d 2>&1 | tail -1)"
    done
  done
done

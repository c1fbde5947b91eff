# K-PRED gather-mode geometry A/B on a shuffled cfg3 batch (tools/gather_ab.py)
out=gpurun_out/r02_gather_ab2.jsonl
: > $out
GNB_ROWGATHER=0 python tools/gather_ab.py gather4 >> $out 2>&1
GNB_RG_NW=1 GNB_RG_CTAS=4 python tools/gather_ab.py nw1_c4 >> $out 2>&1
GNB_RG_NW=2 GNB_RG_CTAS=2 python tools/gather_ab.py nw2_c2 >> $out 2>&1
GNB_RG_NW=2 GNB_RG_CTAS=3 python tools/gather_ab.py nw2_c3 >> $out 2>&1
GNB_RG_NW=4 GNB_RG_CTAS=1 python tools/gather_ab.py nw4_c1 >> $out 2>&1
GNB_RG_NW=4 GNB_RG_CTAS=2 python tools/gather_ab.py nw4_c2 >> $out 2>&1
GNB_RG_NW=4 GNB_RG_CTAS=1 GNB_RG_STAGES=3 python tools/gather_ab.py nw4_c1_s3 >> $out 2>&1
cat $out

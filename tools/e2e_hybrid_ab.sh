# int32 e2e: host narrowing vs hybrid raw-DMA + narrowing chunk splits
python -m pytest tests/test_gpu_predict.py -q -x -p no:cacheprovider -k host 2>&1 | tail -1
for re in 0 2 3 4; do echo raw_every=$re; GNB_HOST_RAW_EVERY=$re GNB_HOST_TIMING=1 python tools/host_read_probe.py 2>&1 | tail -1; done

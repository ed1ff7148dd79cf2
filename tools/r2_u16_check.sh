bash tools/r2_u16_ab.sh
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_ingest.py -m gpu -x -q -k "u16 or sweep or c3_full or c5 or level0 or wide or artifact or session" -p no:warnings 2>&1 | tail -3

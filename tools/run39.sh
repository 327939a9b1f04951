# producerless ring (RB_NOPROD build): parity subset, then A/B timing
RASTERBOUND_B200_LIB=build/ab/noprod.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
bash tools/ab.sh build/ab/cur.so build/ab/noprod.so

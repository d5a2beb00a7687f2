python scratch/dbg_f32.py 2>&1 | tail -8
timeout 900 python -m pytest tests/test_f32tc.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -3
timeout 600 python scratch/f32_time.py 2>&1 | grep tcgen05

timeout 400 python -m pytest tests/test_gpu_comm.py -q -m gpu -x 2>&1 | tail -30
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -4

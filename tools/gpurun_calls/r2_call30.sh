python -m pytest tests/test_gpu_parity.py -k "pinned or profile_iteration" -x -q 2>&1 | tail -3

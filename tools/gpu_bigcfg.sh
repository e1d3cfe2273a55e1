set -x
free -g | head -2
timeout 1800 python -m pytest tests/test_gpu_features.py -m gpu -q -x -k full_size --durations=5 2>&1 | tail -12

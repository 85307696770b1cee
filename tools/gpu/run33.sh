timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "empty or full_size" 2>&1 | tail -8

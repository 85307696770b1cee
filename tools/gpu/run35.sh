timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "shard" 2>&1 | tail -3; timeout 600 python bench.py --steps 5 --warmup 3 --no-table --no-e2e --no-cpu | cut -c1-200

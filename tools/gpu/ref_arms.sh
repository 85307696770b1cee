# both reference arms (CPU only; GPU used to generate the inputs fast)
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 | cut -c1-200
timeout 600 python bench.py --impl reference --workload wave4 --steps 3 --warmup 1

timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "host_runner" 2>&1 | tail -2
for opt in "" "--e2e-no-ramp"; do for c in 12 16 24; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-table --no-cpu --e2e-chunks $c $opt > gpurun_out/b.json 2> gpurun_out/b.err
python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$opt', $c, d['e2e']['value'], d['e2e']['ms_per_step'])"
done; done

timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "shard or wave4" 2>&1 | tail -1
timeout 900 python bench.py --workload wave4 --steps 5 --warmup 3 > gpurun_out/w1.json 2> gpurun_out/w1.err; tail -2 gpurun_out/w1.err
python -c "import json;d=json.load(open('gpurun_out/w1.json'));print('N1', d['value'], d['ms_per_step'], d['scaling'], d['roofline']['frac'], d.get('e2e',{}).get('value'))"

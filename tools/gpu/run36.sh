for opt in "" "--e2e-split-d2h" "--e2e-eager" "--e2e-eager --e2e-split-d2h"; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-table --no-cpu $opt > gpurun_out/b.json 2> gpurun_out/b.err
python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$opt', d['e2e']['value'], d['e2e']['ms_per_step'])"; tail -1 gpurun_out/b.err
done

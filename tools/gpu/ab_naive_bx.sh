timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for bx in 0 256; do
ACS_NAIVE_BX=$bx timeout 600 python bench.py --steps 20 --warmup 3 --no-table --no-e2e --no-cpu --schedule 1 > gpurun_out/b.json 2> gpurun_out/b.err; tail -3 gpurun_out/b.err
python -c "import json;d=json.load(open('gpurun_out/b.json'));print('bx', $bx, d['value'], d['ms_per_step'])"
done

# --workload wave4: N=1 and the N=2 path with both ranks on one GPU (functional only)
mkdir -p gpurun_out
timeout 900 python bench.py --workload wave4 --steps 5 --warmup 3 > gpurun_out/w1.json 2> gpurun_out/w1.err; tail -2 gpurun_out/w1.err
python -c "import json;d=json.load(open('gpurun_out/w1.json'));print('N1', d['value'], d['ms_per_step'], d['scaling'], d['roofline']['frac'], d.get('e2e',{}).get('value'))"
ACS_BENCH_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --workload wave4 --gpus 2 --steps 3 --warmup 3 --size 512 --no-e2e > gpurun_out/w2.json 2> gpurun_out/w2.err; echo "n2 rc=$?"; tail -12 gpurun_out/w2.err
python -c "import json;d=json.load(open('gpurun_out/w2.json'));print('N2', d['value'], d['ms_per_step'], d['config']['grid'])"

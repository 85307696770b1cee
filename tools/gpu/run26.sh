mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "host_runner" > gpurun_out/pytest_hr.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_hr.log
tail -3 gpurun_out/pytest_hr.log
for c in 16 32; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-table --no-cpu --e2e-chunks $c > gpurun_out/bench_e2e_$c.json 2> gpurun_out/bench_e2e_$c.err
python -c "import json;d=json.load(open('gpurun_out/bench_e2e_$c.json'));print($c, d['value'],d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['path'][-40:])"; tail -2 gpurun_out/bench_e2e_$c.err
done

# k-chunk length of the march skeleton (ACS_MARCH_KCHUNK) vs the launcher's automatic choice,
# per march nest: bash tools/gpu/kchunk_sweep.sh > gpurun_out/kchunk.log
mkdir -p gpurun_out
one() {  # kid size dtype sweeps
  for K in ${KS:-0 8 16 24 32 48 64}; do
    ACS_MARCH_KCHUNK=$K timeout 600 python - "$1" "$2" "$3" "$4" "$K" <<'PY'
import json, sys, bench
kid, size, dt, sw, K = sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4]), sys.argv[5]
slot, name, tms = bench.tune_kernel(kid, size, dt, "accsat")
ms, gbs, w = bench.bench_kernel(kid, size, dt, sw, "accsat", "default", reps=5)
print(json.dumps({"kid": kid, "kchunk": K, "slot": slot, "name": name, "gbs": round(gbs, 1),
                  "tms": {k: round(v, 4) for k, v in tms.items()}}), flush=True)
PY
  done
}
if [ "$1" = 2d ]; then   # the 2-D nests around the launcher's minimum chunk
  KS="0 4 6 12"
  for k in swim.c:calc1:0 swim.c:calc2:1; do one $k 8192 f64 1; done
  for k in clover.c:ideal_gas:0 clover.c:pdv_predict:1 clover.c:advec_cell_x:2; do one $k 7680 f64 1; done
  exit 0
fi
one jacobi7.c:jacobi7:0 256 f64 100
one wave4.c:wave4:0 1024 f32 1
one clover.c:pdv_predict:1 7680 f64 1
one swim.c:calc2:1 8192 f64 1

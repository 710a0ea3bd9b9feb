#!/bin/bash
# Gaussian-CRT products: parity tests, per-product timing, refinement A/B.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ozaki.py -x -q > gpurun_out/g_ozaki_tests.log 2>&1; echo ozaki_tests $?
tail -3 gpurun_out/g_ozaki_tests.log
timeout 300 python tools/oz_product_bench.py 8192 5 2>&1 | tail -8
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g_gpu_tests.log 2>&1; echo gpu_tests $?
tail -3 gpurun_out/g_gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err; echo bench $?
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --gemm ozaki_std > gpurun_out/g_bench_std.json 2>> gpurun_out/g_bench.err; echo bench_std $?
python - <<'PY'
import json
for f in ("gpurun_out/g_bench.json", "gpurun_out/g_bench_std.json"):
    try:
        d = json.load(open(f))
        print(f, d["value"], d["result"]["iterations"], d["result"]["final_relE"], d["result"]["final_ortho"], d["roofline"]["share_of_step"], d["roofline"]["achieved"], d["e2e"]["value"])
    except Exception as e:
        print(f, "ERR", e)
PY

#!/bin/bash
# full GPU suite + default bench line + ncu of one Gaussian encode and decode
mkdir -p gpurun_out
tag=${1:-chk}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gpu_tests.log 2>&1; echo gpu_tests $?; tail -1 gpurun_out/${tag}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench $?
python -c "import json; d=json.load(open('gpurun_out/${tag}_bench.json')); print(d['value'], d['result']['iterations'], d['result']['final_relE'], d['result']['final_ortho'], d['roofline']['share_of_step'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'], d['gpu_launches'])"
if [ -n "$2" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"encode_kernel|decode_kernel" --launch-skip 34 --launch-count 3 \
  -o gpurun_out/${tag}_encdec -f python tools/oz_product_bench.py 8192 1 > gpurun_out/${tag}_ncu_encdec.log 2>&1; echo ncu $?
fi

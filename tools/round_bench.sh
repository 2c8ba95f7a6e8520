#!/bin/bash
# A round's evidence in one gpurun call: smoke, the GPU test suite, bench lines
# of configs 0-3 (driver defaults), the reference arm, the one-rank NCCL data
# path through bench.py.  Outputs in gpurun_out/.
set -u
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 > $O/gpu_tests.log 2>&1
echo "pytest rc=$?" >> $O/gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err
for c in c3 c1 c0; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --dp-one-rank --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_dp1.json 2> $O/bench_dp1.err

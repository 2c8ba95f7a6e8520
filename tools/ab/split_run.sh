O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_solver.py tests/test_gpu_rows.py tests/test_gpu_projector.py tests/test_gpu_binding.py -q -x > $O/t_split.log 2>&1
for f in 1 0 1; do PT_GATHER_SPLIT=$f timeout 600 python bench.py --config c0 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/bench_c0_split$f.json 2>&1; python -c "
import json
d=json.loads(open('$O/bench_c0_split$f.json').read().strip().splitlines()[-1])
print('split $f', d['value'], d['kernel_times']['snap_gather'], d['kernel_times']['snapshot'])" >> $O/split_times.txt; done

O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fgp.py tests/test_gpu_rows.py -q -x > $O/t_small.log 2>&1
for c in c0 c1; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done

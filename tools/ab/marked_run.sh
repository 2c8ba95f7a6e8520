O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -rf > $O/t_marked.log 2>&1; echo "rc=$?" >> $O/t_marked.log
for c in c0 c1; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done

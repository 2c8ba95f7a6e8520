O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_solver.py tests/test_gpu_binding.py -q -x > $O/t_fuse.log 2>&1
for f in 1 0 1; do PT_FUSE_REDUCE=$f timeout 600 python bench.py --config c0 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/bench_c0_fuse$f.json 2>&1; done

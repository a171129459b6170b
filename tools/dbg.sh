python -c "import __graft_entry__ as g; g.build()" > gpurun_out/dbg_build.log 2>&1
timeout 300 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -k breakdown -x -q > gpurun_out/dbg_cs1.log 2>&1
for n in 16 40 96 200 384; do timeout 120 python bench.py --n $n --steps 2 --warmup 3 --no-e2e --no-csr --no-cpu > gpurun_out/dbg_b$n.json 2> gpurun_out/dbg_b$n.err; echo "n=$n rc=$?"; done
timeout 300 compute-sanitizer --tool memcheck python bench.py --n 40 --steps 2 --warmup 3 --no-e2e --no-csr --no-cpu > gpurun_out/dbg_cs2.log 2>&1

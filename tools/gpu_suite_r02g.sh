#!/bin/bash
# round-2 final suite + GPU tests + e2e copy-rate probe. Usage: bash tools/gpu_suite_r02g.sh TAG
TAG=${1:-r02g}; OUT=gpurun_out/$TAG; mkdir -p $OUT
bash tools/gpu_tests.sh $TAG > /dev/null 2>&1; tail -3 $OUT/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log; tail -2 $OUT/smoke.log
python - > $OUT/pcie.txt 2>&1 <<'P'
import torch, time
n = 171199875
h = torch.empty(n, dtype=torch.float64).pin_memory(); d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, f in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    f(); torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(3): f()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
    print(name, "%.1f GB/s" % (n * 8 / dt / 1e9))
P
cat $OUT/pcie.txt
bash tools/run_bench_suite.sh $TAG

# co-resident TMA kernel: new default (2 x 64 KB, variant 0) vs the first default (3 x 32 KB, variant 6), alternating
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_tma.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_tma.log
python -c "import __graft_entry__ as g; g.smoke()" && echo smoke ok
for c in 8 4 2 16; do
for rep in 1 2; do
for v in 0 6; do
  RAVNEST_B200_TMA_VARIANT=$v timeout 300 python bench.py --steps 50 --warmup 5 --clusters $c --cpu-sample-params 200000 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bert C=$c variant $v', d['ms_per_step'], d['avg_kernel_ms'], d['roofline']['frac'], d.get('clocks'))"
done; done; done

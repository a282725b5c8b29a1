# co-resident TMA kernel: stage size / count variants at N=1 (BERT, ResNet-50)
for wl in bert resnet50; do
for v in 6 8 9 10 11 6 0; do
  RAVNEST_B200_TMA_VARIANT=$v timeout 300 python bench.py --steps 50 --warmup 5 --workload $wl 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl variant $v', d['ms_per_step'], d['avg_kernel_ms'], d['roofline']['frac'], d.get('clocks',{}).get('sm_mhz'))"
done; done

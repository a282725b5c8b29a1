# A/B of two builds of the library on one GPU (tools/_ab/{old,new}.so, git-ignored), N=1
LIB=paper_2401_01728_b200/libravnest_b200.so
cp $LIB tools/_ab/keep.so
for wl in bert resnet50; do for rep in 1 2 3; do for v in new old; do
  cp tools/_ab/$v.so $LIB
  timeout 300 python bench.py --workload $wl --steps 50 --cpu-sample-params 100000 --ref-sample-params 100000 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl $v', d['ms_per_step'], d['avg_kernel_ms'], d['roofline']['frac'])"
done; done; done
cp tools/_ab/keep.so $LIB

# e2e (host buffers through rv_allreduce_mean_host) at N=1: pipeline lanes
for rep in 1 2; do for l in 16 32 64; do
  timeout 300 python bench.py --steps 20 --e2e-lanes $l --cpu-sample-params 100000 --ref-sample-params 100000 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('e2e lanes $l', d['e2e']['value'], d['e2e']['ms_per_step'])"
done; done

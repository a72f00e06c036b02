# Dev tool: bench at N GPUs, NCCL all-reduce vs NVLink owner-gather exchange, interleaved
N=${1:-2}
for r in 1 2; do for m in nccl nvl; do
  PPMOE_TP_COMM=$m timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29$((700+r*10+${#m})) bench.py --gpus $N --steps 20 --warmup 3 --no-e2e --no-a2a 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$N $m', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done

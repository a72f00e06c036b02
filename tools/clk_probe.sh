for m in off nvml smi; do for c in nvl nccl; do
PPMOE_CLOCKS=$m PPMOE_TP_COMM=$c timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29$((600+${#m}*10+${#c})) bench.py --gpus 4 --steps 20 --warmup 3 --no-a2a --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('clocks=$m comm=$c', round(d['value']), round(d['ms_per_step'],3), d['clocks'])"
done; done

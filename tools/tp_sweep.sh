# TP overlap sweep (dev tool): bench at N GPUs over forward chunking x GEMM SM budget
N=${1:-4}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | grep -E "FAILED|Error|passed|failed" | head -8
for c in 1 4; do for b in 148 132 116; do
  PPMOE_FWD_CHUNKS=$c PPMOE_OVERLAP_SMS=$b timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29$((500+c*10+b%100)) bench.py --gpus $N --steps 20 --warmup 3 --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$N chunks=$c sms=$b', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"
done; done

run() { timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 500)) tools/nvl_micro.py "$@" 2>&1 | grep '^\[T' | sort; }
for E in 4 8; do
run $E
PPMOE_OG_CTAS=8 run $E
PPMOE_OG_FWD_CW=8 run $E
PPMOE_NVL_PULL=sm run $E
PPMOE_NVL_PUSH=1 PPMOE_NVL_PULL=sm run $E
PPMOE_NVL_FWD=fused run $E
done

#!/bin/bash
# Under torch.distributed.run --no-python: rank 0 runs the given python command under ncu with
# the NVLink / DRAM counters of the exchange kernels (single-GPU capture of a multi-rank job:
# only rank 0's kernels are replayed; its peers wait at the next barrier), other ranks plain.
#   python -m torch.distributed.run --nproc-per-node 2 --no-python tools/ncu_rank0.sh OUT.csv tools/nvl_micro.py 8 3
out="$1"; shift
if [ "${RANK:-0}" = "0" ]; then
  exec ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:"nvl_owner_gather|nvl_pull_blocks" -c 8 --csv --log-file "$out" python "$@"
else
  exec python "$@"
fi

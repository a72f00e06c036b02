#!/bin/bash
# Under torch.distributed.run --no-python: every rank runs the given python command under
# compute-sanitizer (tool from $SANITIZER_TOOL, default memcheck), log per rank.
#   python -m torch.distributed.run --nproc-per-node 2 --no-python tools/sanitize_rank.sh PREFIX tools/nvl_micro.py 8 2
pre="$1"; shift
exec compute-sanitizer --tool "${SANITIZER_TOOL:-memcheck}" --print-limit 50 --log-file "${pre}.rank${RANK:-0}.log" python "$@"

# Final-evidence pass on 4 GPUs: multi-rank suite, bench lines at T = 4 (C2, C3) and T = 2.
set -x
timeout 1500 python -m pytest tests/test_gpu_multirank.py -m gpu -q -x > gpurun_out/mr4.log 2>&1; tail -2 gpurun_out/mr4.log
timeout 500 python bench.py --gpus 4 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; tail -1 gpurun_out/bench4.json | cut -c1-200
timeout 700 python bench.py --gpus 4 --config c3 > gpurun_out/bench4c3.json 2> gpurun_out/bench4c3.err; tail -1 gpurun_out/bench4c3.json | cut -c1-200
CUDA_VISIBLE_DEVICES=0,1 timeout 500 python bench.py --gpus 2 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -1 gpurun_out/bench2.json | cut -c1-200

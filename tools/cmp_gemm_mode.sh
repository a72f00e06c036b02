# per-GEMM comparison of the 1-CTA and CTA-pair kernels inside the C2 step (dev tool)
mkdir -p gpurun_out
python tools/prof_step.py > gpurun_out/plain.log 2>&1 || exit 1
PPMOE_GEMM=single python tools/prof_step.py >> gpurun_out/plain.log 2>&1 || exit 1
for m in single pair; do
  PPMOE_GEMM=$m timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file gpurun_out/mode_$m.csv python tools/prof_step.py > /dev/null 2>&1
done
for m in single pair; do
  PPMOE_GEMM=$m timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['achieved']), d['clocks']['sm_mhz'], {k[13:]: v['ms_per_step'] for k, v in d['kernels'].items() if 'expert' in k})"
done

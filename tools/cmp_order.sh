# A/B of GEMM scheduling/caching options on the C2 step (dev tool)
mkdir -p gpurun_out
python tools/prof_step.py > gpurun_out/plain.log 2>&1 || exit 1
for v in "PPMOE_STORE=normal" "PPMOE_STORE=cs" "PPMOE_STORE=cs PPMOE_HINT=1" "PPMOE_STORE=normal PPMOE_HINT=1"; do
  env $v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), round(d['ms_per_step'],3), round(d['roofline']['achieved']), d['clocks']['sm_mhz'])"
done
for v in "PPMOE_STORE=normal" "PPMOE_STORE=cs PPMOE_HINT=1"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file gpurun_out/l_$tag.csv python tools/prof_step.py > /dev/null 2>&1
done

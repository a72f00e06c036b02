# Final-evidence pass on one GPU: GPU suite, smoke, bench lines (C2, C3, reference arm), the
# ncu launch list of the C2 step. Outputs under gpurun_out/.
set -x
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu1.log 2>&1; tail -2 gpurun_out/gpu1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -1 gpurun_out/bench1.json | cut -c1-200
timeout 600 python bench.py --config c3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -1 gpurun_out/bench_c3.json | cut -c1-200
timeout 400 python bench.py --impl reference > gpurun_out/ref.json 2> gpurun_out/ref.err; tail -1 gpurun_out/ref.json | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 150 --csv --log-file gpurun_out/launch_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-a2a > gpurun_out/ncu_c2.log 2>&1; tail -1 gpurun_out/ncu_c2.log | cut -c1-100

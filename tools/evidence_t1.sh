set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 400 python bench.py --impl reference > gpurun_out/ref.json 2> gpurun_out/ref.err; tail -1 gpurun_out/ref.json | cut -c1-300
timeout 600 python bench.py --config c3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -1 gpurun_out/bench_c3.json | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 150 --csv --log-file gpurun_out/launch_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-a2a > gpurun_out/ncu_c2.log 2>&1; tail -1 gpurun_out/ncu_c2.log | cut -c1-100
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 150 --csv --log-file gpurun_out/launch_c3.csv python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-a2a > gpurun_out/ncu_c3.log 2>&1; tail -1 gpurun_out/ncu_c3.log | cut -c1-100
timeout 300 ncu --set full --import-source on --clock-control none -k regex:router_tc_kernel -s 2 -c 1 -o gpurun_out/r02_router_tc_full python tools/prof_router.py > gpurun_out/tcfull.log 2>&1; tail -1 gpurun_out/tcfull.log

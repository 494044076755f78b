set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err; tail -c 600 gpurun_out/bench_g.json
timeout 120 python tools/bwd_time.py 8192 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -s 6 -c 6 python tools/bwd_time.py 8192 > gpurun_out/bwd_launches.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bwd_pair -s 2 -c 2 -o gpurun_out/prof_bwdpair3 python tools/bwd_time.py 8192 > gpurun_out/ncu_bwdpair3.log 2>&1; tail -1 gpurun_out/ncu_bwdpair3.log

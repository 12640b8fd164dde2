timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
timeout 300 python tools/bench_build.py > gpurun_out/build.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ncu_build.csv python tools/bench_build.py --profile > gpurun_out/ncu_build.log 2>&1

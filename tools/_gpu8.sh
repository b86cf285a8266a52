timeout 900 ncu --set full --clock-control none --import-source on -k regex:gmt_solve_kernel -c 3 -o gpurun_out/di_solve -f python tools/di_batch_ncu.py > gpurun_out/ncu_di.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --forest-queries 0 --e2e-steps 2 > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 600 python tools/scale_probe.py > gpurun_out/scale.log 2>&1; tail -4 gpurun_out/scale.log

mkdir -p gpurun_out
timeout 900 python scripts/calibrate_decode_cost.py > gpurun_out/calib.log 2>&1; echo calib=$?; tail -5 gpurun_out/calib.log

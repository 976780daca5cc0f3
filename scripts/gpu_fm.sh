timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_configs.py -q -x 2>&1 | tail -2
AB='{"base":{}}' CASES=FP8_E4M3:1:16,FP8_E4M3:8:16,FP8_E4M3:8:256,FP8_E4M3:16:512,FP16:8:16,INT4:8:32,INT4:64:64,FP8_E4M3:16:2048 timeout 600 python scripts/ab_decode.py 2>&1 | grep -E "GB/s|Error" | head

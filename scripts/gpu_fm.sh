AB='{"iq":{}, "pk":{"KVSLAB_DECODE_PACK":"3"}}' CASES=INT4:32:112,INT4:8:256,INT4:16:512,INT4:16:2048 timeout 600 python scripts/ab_decode.py 2>&1 | grep -E "GB/s|Error" | head

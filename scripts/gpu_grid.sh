C=""
for f in FP16 FP8_E4M3 INT8 INT4; do for b in 1 4 16 64; do for c in 1024 4096 16384; do
  if [ $((b * c)) -le 262144 ]; then C="$C,$f:$b:$c"; fi
done; done; done
C=${C#,}
AB='{"r02":{}}' CASES=$C ROUNDS=3 timeout 1200 python scripts/ab_decode.py 2>&1 | grep -E "GB/s|Error"

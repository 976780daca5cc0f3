# ncu evidence for profiles/: launch list of one bench step + full capture of K2
set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'paged_decode|merge_kernel|table_scatter' --csv --log-file gpurun_out/launches.csv python bench.py --profile > gpurun_out/prof_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'paged_decode|merge_kernel' -c 4 -o gpurun_out/decode_full -f python bench.py --profile > gpurun_out/prof_full.log 2>&1; echo ncu2=$?
ls -la gpurun_out

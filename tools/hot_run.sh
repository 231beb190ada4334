#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"nmf_wpass" -s 4 -c 4 --csv --log-file gpurun_out/hot_nmf_t.csv python tools/time_gnmf.py > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"kmeans_pass" -s 4 -c 4 --csv --log-file gpurun_out/hot_km_t.csv python tools/time_kmeans.py > /dev/null 2>&1
grep -v "^==" gpurun_out/hot_nmf_t.csv | awk -F'","' '{print $5" "$(NF-2)" "$(NF-1)" "$NF}' | cut -c1-160
grep -v "^==" gpurun_out/hot_km_t.csv | awk -F'","' '{print $5" "$(NF-2)" "$(NF-1)" "$NF}' | cut -c1-160
for i in 1 2 3; do timeout 300 python tools/time_gnmf.py; done

#!/bin/bash
# L2 / fabric / DRAM counters of the bench's task kernel per library variant.
M=dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_requests_srcunit_ltcfabric.sum,lts__t_requests_srcunit_ltcfabric_lookup_miss.sum,lts__d_sectors_fill_device.sum,gpu__time_duration.sum
for v in "$@"; do
  TILEMUL_B200_LIB=$PWD/exp_libs/$v.so timeout 900 ncu --metrics $M --clock-control none -k "regex:k_dmma($|<)" -s 3 -c 1 --csv \
    --log-file gpurun_out/l2_$v.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
  echo "== $v rc=$?"
  grep -E '"k_dmma|k_dmma' gpurun_out/l2_$v.csv | awk -F'","' '{print $(NF-2), $NF}'
done

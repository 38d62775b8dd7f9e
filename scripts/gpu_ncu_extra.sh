# extra ncu evidence (VERDICT weak #12): k/v GEMM, the gather, the stream-K merged-code decode GEMV
# (down projection, T = 4) and the down-projection router (h = 3584, T = 8192), plus their launch lists
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mobi_gemm_tc2 -s 6 -c 1 -o gpurun_out/x_kv_gemm -f $B --out 1024 --in 4096 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/x_kv_launches.csv $B --out 1024 --in 4096 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather_kernel -s 6 -c 1 -o gpurun_out/x_gather -f $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_gemm_kernel -s 4 -c 1 -o gpurun_out/x_down_dec -f $B --out 4096 --in 14336 --tokens 4 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/x_down_dec_launches.csv $B --out 4096 --in 14336 --tokens 4 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:router_tc -s 3 -c 1 -o gpurun_out/x_down_router -f $B --out 4096 --in 14336 --tokens 8192 --ring 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/x_down_launches.csv $B --out 4096 --in 14336 --tokens 8192 --ring 1 > /dev/null 2>&1
ls -la gpurun_out/x_*

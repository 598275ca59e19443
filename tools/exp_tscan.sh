cd $GRAFT_REPO_ROOT
for T in 2048 4096 8192 16384; do FFWD_LIB=build/libffwd_probe.so timeout 300 python tools/probe_gemm.py 8b $T 2>&1 | grep "T="; done
for T in 4096 16384; do
FFWD_T=$T timeout 600 ncu --clock-control none -k regex:down_proj -s 2 -c 1 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_read.sum python tools/prof_layer.py 8b 3 sparse 2>&1 | grep -E "down_proj|dram__|lts__|tensor|duration" 
FFWD_T=$T timeout 600 ncu --clock-control none -k regex:up_proj -s 2 -c 1 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active python tools/prof_layer.py 8b 3 sparse 2>&1 | grep -E "up_proj|dram__|lts__|tensor|duration" 
done

M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_requests.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,smsp__inst_executed.sum,l1tex__m_xbar2l1tex_read_sectors.sum,l1tex__data_pipe_lsu_wavefronts_mem_lg.sum,l1tex__t_sector_hit_rate.pct,smsp__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed,l1tex__lsu_writeback_active_mem_lg.sum,lts__t_sectors_srcunit_tex.sum
for sa in $STOPS; do
  echo "== stop $sa"
  GK_STOP_AFTER=$sa ncu --metrics $M --clock-control none -k regex:bfs_persistent -s 0 -c 1 --csv python tools/ncu_one.py --config $CFG --runs 1 2>/dev/null | grep -v "^==" | grep bfs_persistent | awk -F'","' '{print $(NF-2), $NF}'
done

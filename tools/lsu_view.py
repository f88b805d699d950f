"""LSU data-pipe view of an ncu raw CSV (ncu -i rep --page raw --csv): wavefronts by
memory space, sectors, bytes per sector access, bank conflicts, per kernel launch."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, data = rows[0], rows[2:]
def col(name):
    return [r[h.index(name)] for r in data] if name in h else None
names = col('Kernel Name')
pick = ['gpu__time_duration.sum', 'launch__grid_size',
        'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
        'SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg',
        'SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_shared.avg',
        'SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_st.sum',
        'smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio',
        'smsp__sass_average_data_bytes_per_sector_mem_global_op_st.ratio',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__sass_inst_executed_op_ldgsts_cache_access.sum', 'smsp__inst_executed_op_ldgsts.sum',
        'smsp__sass_l1tex_data_pipe_lsu_wavefronts_mem_shared_op_ldgsts.sum']
print('kernels:', [n[:28] for n in names])
for p in pick:
    c = col(p)
    if c:
        print(p.ljust(84), c)

# Compose a profiles/ summary of one ncu --set full report:
#   bash tools/profile_summary.sh REPORT UNITS "header line" > profiles/X.txt
rep=$1; units=$2
echo "# $3"
echo "## headline + stalls + SASS opcode mix per unit (tools/ncu_summary.py)"
python tools/ncu_summary.py "$rep" "$units"
echo
echo "## pipe utilisation (% of peak, active cycles)"
ncu -i "$rep" --page raw --csv 2>/dev/null | python -c "
import csv, sys
rows = list(csv.reader(sys.stdin)); h, v = rows[0], rows[2]
for i, k in enumerate(h):
    if (k.startswith('sm__inst_executed_pipe_') or k.startswith('sm__pipe_')) and k.endswith('avg.pct_of_peak_sustained_active'):
        try:
            if float(v[i]) > 0.5: print(f'  {k:80s} {float(v[i]):8.2f}')
        except ValueError:
            pass
for k in ('sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed',
          'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed'):
    if k in h: print(f'  {k:80s} {float(v[h.index(k)]):8.2f}')
"
echo
echo "## instructions per unit by CUDA source line (tools/ncu_srcmix.py; inlined helpers double-count their callers)"
python tools/ncu_srcmix.py "$rep" "$units" 30
echo
echo "## stall samples by opcode (tools/ncu_stalls.py)"
python tools/ncu_stalls.py "$rep" 20

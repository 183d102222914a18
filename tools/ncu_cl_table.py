"""Print the per-kernel table of a tools/cl_iter.sh ncu CSV: python tools/ncu_cl_table.py file.csv [regex]."""
import collections
import csv
import re
import sys

rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else "k_cl_count|k_cl_fill")
hdr = rows[0]
ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
d = collections.OrderedDict()
for r in rows[1:]:
    d.setdefault((r[ii], r[ki]), {})[r[mi]] = r[vi]
for (i, k), m in d.items():
    if not pat.search(k):
        continue
    g = lambda n: float(m.get(n, "0").replace(",", ""))  # noqa: E731
    name = re.sub(r"\(.*", "", k).split("::")[-1]
    print(f"{name:22s} {g('gpu__time_duration.sum') / 1e3:9.1f} us  inst {g('smsp__inst_executed.sum') / 1e6:8.1f}M  "
          f"issue {g('smsp__issue_active.avg.pct_of_peak_sustained_elapsed'):5.1f}%  "
          f"lsu wavefronts {g('l1tex__data_pipe_lsu_wavefronts.sum') / 1e6:8.1f}M ({g('l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed'):4.1f}%)  "
          f"warps {g('sm__warps_active.avg.pct_of_peak_sustained_active'):4.1f}%  "
          f"gld sectors {g('l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum') / 1e6:8.1f}M  L2 rd sectors {g('lts__t_sectors_srcunit_tex_op_read.sum') / 1e6:8.1f}M  "
          f"dram R {g('dram__bytes_read.sum') / 1e9:6.2f} W {g('dram__bytes_write.sum') / 1e9:6.2f} GB")

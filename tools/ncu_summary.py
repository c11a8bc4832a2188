"""Summarise ncu reports: key throughput / memory metrics per kernel.

    python tools/ncu_summary.py report.ncu-rep [...]   (prints a table)
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "dur"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "ld_sect"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "ld_req"),
    ("l1tex__t_sector_hit_rate.pct", "l1hit%"),
    ("lts__t_sectors.sum", "l2_sect"),
    ("lts__t_requests.sum", "l2_req"),
    ("lts__t_sector_hit_rate.pct", "l2hit%"),
    ("lts__t_sectors_srcunit_ltcfabric.sum", "fabric"),
    ("lts__t_sectors_op_red.sum", "l2_red_sect"),
    ("lts__t_sectors_op_atom.sum", "l2_atom_sect"),
    ("l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed", "xbar_req%"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum", "red_sect"),
    ("smsp__inst_executed_op_global_red.sum", "red_inst"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("smsp__inst_executed.sum", "inst"),
    ("launch__registers_per_thread", "regs"),
]


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    for row in r[2:]:
        d = {"kernel": row[h.index("Kernel Name")][:48]}
        for k, short in KEYS:
            if k in h:
                d[short] = (row[h.index(k)], units[h.index(k)])
        yield d


if __name__ == "__main__":
    for p in sys.argv[1:]:
        for d in rows(p):
            print(p.split("/")[-1], d["kernel"])
            print("   " + "  ".join(f"{k}={v[0]}{v[1] if v[1] not in ('', 'sector', 'request', 'inst') else ''}"
                                  for k, v in d.items() if k != "kernel"))

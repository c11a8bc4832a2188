"""Build profiles/ncu_summary.json (read by bench.py) from the raw-page CSV
exports of the round's --set full captures of one encode step (tools/
gpu_prof_r02.sh): per pass (all launches of fh_encode_fwd / fh_encode_bwd_ex
of the LAST captured step) the durations, DRAM bytes, and the time-weighted
L2 / L1->XBAR utilisation.

    python tools/make_ncu_summary.py gpurun_out/r02_encode_cfg2_raw.csv gpurun_out/r02_encode_cfg4_raw.csv
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M = {
    "dur": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "lts": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "xbar": "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "red_sect": "lts__t_sectors_srcunit_tex_op_red.sum",
    "red_pct": "lts__t_sectors_srcunit_tex_op_red.avg.pct_of_peak_sustained_elapsed",
    "atom_in": "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l2hit": "lts__t_sector_hit_rate.pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1,
         "msecond": 1e3, "ms": 1e3}


def launches(path):
    r = list(csv.reader(open(path)))
    h, u = r[0], r[1]
    out = []
    for row in r[2:]:
        d = {"kernel": row[h.index("Kernel Name")].split("(")[0]}
        for k, m in M.items():
            if m in h:
                v = float(row[h.index(m)].replace(",", "") or 0)
                d[k] = v * SCALE.get(u[h.index(m)], 1)
        out.append(d)
    return out


def last_step(ls):
    """The last fwd run followed by its bwd run."""
    i = len(ls) - 1
    while i >= 0 and "fwd_kernel" not in ls[i]["kernel"]:
        i -= 1
    j = i
    while j > 0 and "fwd_kernel" in ls[j - 1]["kernel"]:
        j -= 1
    return ls[j:i + 1], ls[i + 1:]


def summarise(ls):
    t = sum(x["dur"] for x in ls)
    w = lambda k: sum(x[k] * x["dur"] for x in ls) / t / 100.0
    return {"launches": [x["kernel"] for x in ls], "duration_us": [round(x["dur"], 1) for x in ls],
            "dram_bytes": int(sum(x["dram_rd"] + x["dram_wr"] for x in ls)),
            "dram_read_bytes": int(sum(x["dram_rd"] for x in ls)), "dram_write_bytes": int(sum(x["dram_wr"] for x in ls)),
            "lts_throughput_frac": round(w("lts"), 3), "l1tex2xbar_req_frac": round(w("xbar"), 3),
            "l2_red_sectors": int(sum(x["red_sect"] for x in ls)), "l2_red_rate_frac": round(w("red_pct"), 3),
            "l2_atomic_input_frac": round(w("atom_in"), 3), "l2_hit_frac": round(w("l2hit"), 3)}


def main():
    out = {"_source": "ncu --set full --clock-control none of tools/time_encode.py <cfg> 1 (FH_OVERWRITE=1) on one "
                      "B200, round 2 (tools/gpu_prof_r02c_encode.sh); per encode PASS = all launches of fh_encode_fwd / "
                      "fh_encode_bwd_ex of the last captured step.  *_frac = time-weighted fraction of the unit's "
                      "peak (lts__throughput, l1tex2xbar request port, L2 red-sector rate, atomic input).  Cold "
                      "cache, serialised launches: shares, not absolute times, match the bench."}
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(path):   # merge: entries of earlier captures stay unless re-captured
        prev = json.load(open(path))
        prev.update({k: v for k, v in out.items()})
        out = prev
    for p in sys.argv[1:]:
        # cfg4lm: the cfg4 step in the train step's form (level-major dout, tools/gpu_prof_r02d.sh)
        name = "cfg4_lm" if "cfg4lm" in p else "cfg4" if "cfg4" in p else "cfg2"
        fwd, bwd = last_step(launches(p))
        f, b = summarise(fwd), summarise(bwd)
        out[name] = {"source": "profiles/" + os.path.basename(p).replace("_raw.csv", ".txt"), "fwd": f, "bwd": b,
                     "dram_bytes_per_pass": {"fwd": f["dram_bytes"], "bwd": b["dram_bytes"]},
                     "lts_throughput_frac": {"fwd": f["lts_throughput_frac"], "bwd": b["lts_throughput_frac"]},
                     "l1tex2xbar_req_frac": {"fwd": f["l1tex2xbar_req_frac"], "bwd": b["l1tex2xbar_req_frac"]},
                     "l2_red_sectors_per_pass": b["l2_red_sectors"],
                     "l2_hit_frac": {"fwd": f["l2_hit_frac"], "bwd": b["l2_hit_frac"]}}
    with open(path, "w") as fo:
        json.dump(out, fo, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

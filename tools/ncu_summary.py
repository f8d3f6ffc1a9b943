"""Summarise `ncu --page raw --csv` exports (one or more launches per file):
duration, DRAM bytes and rate, tensor-pipe activity, occupancy, registers
and the top warp-stall reasons.  Usage: python tools/ncu_summary.py a.raw.csv ..."""
import csv
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_read"),
        ("dram__bytes_write.sum", "dram_write"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
        ("lts__t_sector_hit_rate.pct", "l2_hit_%"), ("launch__grid_size", "grid"),
        ("launch__registers_per_thread", "regs")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1}

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    for x in rows[2:]:
        print(f"{path.split('/')[-1]}: {x[h.index('Kernel Name')][:90]}")
        vals = {}
        for k, name in KEYS:
            if k in h:
                i = h.index(k)
                vals[name] = (x[i], units[i])
                print(f"    {name:16s} {x[i]} {units[i]}")
        try:
            t = float(vals["time"][0]) * SCALE[vals["time"][1]]
            b = (float(vals["dram_read"][0]) * SCALE[vals["dram_read"][1]] +
                 float(vals["dram_write"][0]) * SCALE[vals["dram_write"][1]])
            print(f"    {'dram_rate':16s} {b / t / 1e9:.0f} GB/s")
        except (KeyError, ValueError, ZeroDivisionError):
            pass
        st = []
        for i, c in enumerate(h):
            if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued"):
                try:
                    st.append((float(x[i]), c.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        st.sort(reverse=True)
        tot = sum(v for v, _ in st) or 1
        print("    stalls          " + " ".join(f"{c}:{v / tot:.2f}" for v, c in st[:5]))

"""Summarise ncu --set full reports (ncu -i <rep> --page raw --csv) into the
metrics the DESIGN / bench cite: duration, SM clock, DRAM bytes, L2 hit rate,
tensor-pipe activity, achieved occupancy, issue activity, top stall reasons.
Usage: python tools/ncu_summary.py report.ncu-rep [...]  -> markdown table on stdout."""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active", "tensor (imma) active %"),
    ("sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active", "tensor (hmma) active %"),
    ("sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "uniform pipe %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
]


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, data = r[0], r[1], r[2:]
    return hdr, units, data


def main(paths):
    for path in paths:
        hdr, units, data = rows(path)
        print("### %s\n" % path.split("/")[-1])
        ki = hdr.index("Kernel Name")
        cols = ["kernel"] + [lab for m, lab in WANT if m in hdr]
        print("| " + " | ".join(cols) + " |")
        print("|" + "---|" * len(cols))
        for d in data:
            vals = [d[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")[:40]]
            for m, lab in WANT:
                if m in hdr:
                    i = hdr.index(m)
                    vals.append("%s %s" % (d[i], units[i]) if units[i] else d[i])
            print("| " + " | ".join(vals) + " |")
        print()


if __name__ == "__main__":
    main(sys.argv[1:])

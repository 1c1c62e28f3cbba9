"""One line per captured launch from an ncu report (raw page): time, throughput, DRAM / L2
traffic, occupancy, tensor-pipe activity, top warp-stall reasons."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
units = rows[1]
col = {h: i for i, h in enumerate(hdr)}
TO_MB = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def g(r, k, scale=1.0, fmt="{:.1f}"):
    i = col.get(k)
    if i is None or not r[i]:
        return "-"
    try:
        return fmt.format(float(r[i].replace(",", "")) * scale)
    except ValueError:
        return r[i]


stall_keys = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")]
print(f"{'kernel':34s} {'us':>7s} {'SM%':>5s} {'Mem%':>5s} {'DRAMrd MB':>9s} {'DRAMwr MB':>9s} {'L2hit%':>6s} "
      f"{'warps%':>6s} {'TC%':>5s}  top stalls")
for r in rows[2:]:
    name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("skg::", "")[:34]
    st = []
    for k in stall_keys:
        try:
            st.append((float(r[col[k]].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
    tot = sum(v for v, _ in st) or 1.0
    top = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(st, reverse=True)[:3])
    print(f"{name:34s} {g(r, 'gpu__time_duration.sum', 1e-3 if False else 1.0):>7s} "
          f"{g(r, 'sm__throughput.avg.pct_of_peak_sustained_elapsed'):>5s} "
          f"{g(r, 'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed'):>5s} "
          f"{g(r, 'dram__bytes_read.sum', TO_MB.get(units[col['dram__bytes_read.sum']], 1e-6)):>9s} "
          f"{g(r, 'dram__bytes_write.sum', TO_MB.get(units[col['dram__bytes_write.sum']], 1e-6)):>9s} "
          f"{g(r, 'lts__t_sector_hit_rate.pct'):>6s} {g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):>6s} "
          f"{g(r, 'sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active'):>5s}  {top}")

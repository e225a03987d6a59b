"""Key metrics of an ncu --set full report (raw page)."""
import csv, subprocess, sys
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__cycles_active.avg.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second"]
def main(path, out=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = [f"# {path}"]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines.append(f"kernel: {name[:160]}")
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                lines.append(f"  {w} = {vals[i]} {units[i]}")
        extra = [h for h in hdr if "tensor" in h and "pct" in h]
        for h in extra[:12]:
            if h not in WANT:
                i = hdr.index(h); lines.append(f"  {h} = {vals[i]} {units[i]}")
    txt = "\n".join(lines); print(txt)
    if out: open(out, "w").write(txt + "\n")
if __name__ == "__main__":
    main(*sys.argv[1:])

"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list:
per-kernel (demangled, epilogue-resolved) total time, count, share."""
import csv, re, sys, collections

def short(name):
    m = re.search(r"gemm_tn_kernel<(\d+), lemo::Bound<\d+, lemo::(\w+)>", name)
    if m:
        return f"gemm_tn_kernel<{m.group(1)},{m.group(2)}>"
    m = re.search(r"gemm_tn_pair_kernel<(?:lemo::)?Bound<256, (?:lemo::)?(\w+)>", name)
    if m:
        return f"gemm_tn_pair_kernel<{m.group(1)}> (256x256 CTA pair)"
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name)
    return name.replace("lemo::fa::", "").replace("lemo::", "")

def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if not l.startswith("==")]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        rows.append((short(r["Kernel Name"]), v))
    return rows

def main(path, out=None):
    rows = load(path)
    tot = collections.defaultdict(float); cnt = collections.Counter()
    for n, v in rows:
        tot[n] += v; cnt[n] += 1
    T = sum(tot.values())
    lines = [f"# {path}: {len(rows)} launches, {T/1e6:.2f} ms total (serialised, cold-cache ncu timing)",
             f"{'kernel':60s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}"]
    for n in sorted(tot, key=lambda k: -tot[k]):
        lines.append(f"{n:60s} {cnt[n]:8d} {tot[n]/1e6:10.3f} {100*tot[n]/T:6.1f}%")
    txt = "\n".join(lines)
    print(txt)
    if out:
        open(out, "w").write(txt + "\n")

if __name__ == "__main__":
    main(*sys.argv[1:])

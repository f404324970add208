"""Top SASS instructions of an ncu report by warp-stall samples.

    python tools/ncu_hot.py REPORT.ncu-rep [N] [kernel-regex]
Prints samples, the top stall reasons and the instruction."""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv"]
    if len(sys.argv) > 3:
        cmd += ["--kernel-name", f"regex:{sys.argv[3]}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    lines = out.splitlines()
    # skip the kernel-name header line
    body = "\n".join(l for l in lines if not l.startswith('"Kernel Name"'))
    rows = list(csv.reader(io.StringIO(body)))
    h = rows[0]
    idx = {k: i for i, k in enumerate(h)}
    samp = idx["Warp Stall Sampling (All Samples)"]
    stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    tot = sum(float(r[samp] or 0) for r in rows[1:] if len(r) > samp)
    print(f"total samples {tot:.0f}")
    agg = {}
    for r in rows[1:]:
        for s in stalls:
            agg[s] = agg.get(s, 0) + float(r[idx[s]] or 0)
    print("stalls:", ", ".join(f"{k[6:]}={v / tot:.1%}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
    rs = sorted(rows[1:], key=lambda r: -float(r[samp] or 0))[:n]
    for r in rs:
        st = sorted(((float(r[idx[s]] or 0), s[6:]) for s in stalls), reverse=True)[:3]
        print(f"{float(r[samp]):7.0f} {float(r[samp]) / tot:6.1%}  {r[idx['Address']][-5:]}  "
              f"{r[idx['Source']].strip()[:60]:60s} " + " ".join(f"{b}={a:.0f}" for a, b in st if a))


if __name__ == "__main__":
    main()

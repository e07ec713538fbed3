"""Attribute an ncu source-page CSV (SASS view, --print-source sass) of k_layer to CUDA source
lines via nvdisasm -g of the built library: warp-stall samples and top stall reasons per line.

    python tools/ncu_lines.py gpurun_out/X_src.csv [file-filter] [top]
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def addr_lines():
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2601_01310_b200", "libtarragon.so")],
                   cwd=d, capture_output=True)
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, "tg_gemm.sm_100a.cubin")], capture_output=True,
                         text=True).stdout
    out, cur, infn = {}, None, False
    for line in dis.splitlines():
        if line.startswith("//----") and ".text." in line:
            infn = "k_layer" in line
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
        if m and infn and cur:
            out[int(m.group(1), 16)] = cur
    return out


def main():
    path = sys.argv[1]
    filt = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    a2l = addr_lines()
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    H = {h: i for i, h in enumerate(hdr)}
    rc = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    body = [r for r in rows[2:] if r and r[0].startswith("0x")]
    base = int(body[0][0], 16)
    tot, ex, why = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
    for r in body:
        ln = a2l.get(int(r[0], 16) - base, ("?", 0))
        tot[ln] += int(r[H["Warp Stall Sampling (All Samples)"]] or 0)
        ex[ln] += int(r[H["Instructions Executed"]] or 0)
        for c in rc:
            v = r[H[c]]
            if v and v != "0":
                why[ln][c[6:]] += int(float(v))
    allS = sum(tot.values())
    byf = collections.Counter()
    for (f, _), v in tot.items():
        byf[f] += v
    print("samples", allS, "by file", byf.most_common(6))
    sel = [(ln, v) for ln, v in tot.items() if filt in ln[0]]
    for ln, v in sorted(sel, key=lambda x: -x[1])[:top]:
        print(f"{v:7d} {100.0 * v / allS:5.1f}% {ln[0]}:{ln[1]:<5d} exec {ex[ln]:9d}  {why[ln].most_common(3)}")


if __name__ == "__main__":
    main()

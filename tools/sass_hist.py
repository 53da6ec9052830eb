"""SASS opcode histogram of the built library, per kernel family (evidence that the
pipelines issue TMA / bulk copies and mbarrier waits, and how wide the exact rows are).

    python tools/sass_hist.py > profiles/r2_sass_hist.txt
"""
import collections
import os
import re
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(REPO, "paper_2307_00124_b200", "_lib", "libbfpmg_b200.so")
KEY = ["UTMALDG", "UTMASTG", "UBLKCP", "SYNCS", "LDG", "STG", "LDS", "STS", "SHFL", "IMAD",
       "IADD3", "SHF", "LOP3", "ATOMG", "RED", "BAR", "HMMA", "UTCHMMA"]
FAMILY = [("bulk3_win_kernel", "3-D tiled-TMA stencil march"),
          ("bulk_win_kernel", "2-D bulk-copy stencil march"),
          ("pro3_win_kernel", "3-D prolongation march"),
          ("rst3_win_kernel", "3-D restriction march"),
          ("pro2_win_kernel", "2-D prolongation march"),
          ("rst2_win_kernel", "2-D restriction march"),
          ("march_win_kernel", "register march"),
          ("grid_win_kernel", "generic grid kernel"),
          ("coarse_kernel", "persistent coarse-level kernel"),
          ("fused_kernel", "fused single-CTA interpreter"),
          ("dot_", "exact dot"),
          ("", "other")]


def main():
    so = sys.argv[1] if len(sys.argv) > 1 else SO
    txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    fam_ops = collections.defaultdict(collections.Counter)
    fam_n = collections.Counter()
    cur = None
    for ln in txt.splitlines():
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            name = m.group(1)
            cur = next(f for k, f in FAMILY if k in name)
            fam_n[cur] += 1
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", ln)
        if m and cur:
            fam_ops[cur][m.group(2)] += 1
    print(f"# SASS opcode histogram of {os.path.relpath(so, REPO)} (cuobjdump -sass), per kernel "
          "family; counts are static instructions summed over the family's instantiations")
    print("family | functions | " + " | ".join(KEY))
    tot = collections.Counter()
    for _, f in FAMILY:
        if f not in fam_n:
            continue
        tot.update(fam_ops[f])
        print(f"{f} | {fam_n[f]} | " + " | ".join(str(fam_ops[f][k]) for k in KEY))
    print(f"total | {sum(fam_n.values())} | " + " | ".join(str(tot[k]) for k in KEY))


if __name__ == "__main__":
    main()

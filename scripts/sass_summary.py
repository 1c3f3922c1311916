"""Per-kernel SASS instruction summary of the shipped liblcnn_cuda.so: counts
of the Blackwell mnemonics that prove the data paths (tcgen05 MMA / TMEM
loads, TMA tensor loads/stores/reductions, bulk copies, mbarriers) plus
register / spill facts from cuobjdump -res-usage.  Writes
profiles/r02_sass_summary.txt."""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1610_03618_b200", "lib", "liblcnn_cuda.so")
KEYS = ["UTCHMMA", "UTCHMMA.2CTA", "UTCQMMA", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMAREDG",
        "UBLKCP", "UBLKRED", "SYNCS", "MUFU.EX2", "LDG*.128", "STG*.128", "LDGSTS", "HMMA"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    per = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            per[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if not m:
            continue
        op = m.group(1)
        for k in KEYS:
            if op == k or op.startswith(k + "."):
                per[cur][k] += 1
        if op.startswith(("LDG", "STG")) and ".128" in op:
            per[cur][op[:3] + "*.128"] += 1
    demangled = subprocess.run(["c++filt"], input="\n".join(per), capture_output=True,
                               text=True).stdout.splitlines()
    total = collections.Counter()
    lines = [f"SASS summary of {os.path.relpath(LIB, ROOT)} (cuobjdump -sass, sm_100a)", ""]
    for (name, cnt), dem in zip(per.items(), demangled):
        total.update(cnt)
        if not cnt:
            continue
        short = re.sub(r"\(.*", "", dem)[:110]
        lines.append(f"{short}")
        lines.append("    " + ", ".join(f"{k}={cnt[k]}" for k in KEYS if cnt[k]))
    lines.insert(2, "TOTAL: " + ", ".join(f"{k}={total[k]}" for k in KEYS if total[k]))
    lines.insert(3, f"kernels: {len(per)}")
    lines.insert(4, "")
    out = os.path.join(ROOT, "profiles", "r02_sass_summary.txt")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:6]))


if __name__ == "__main__":
    main()

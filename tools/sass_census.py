"""Per-kernel SASS instruction census of libhygen.so (cuobjdump; runs without a GPU).

python tools/sass_census.py [out.md]

For every kernel: registers / shared memory / spills (cuobjdump -res-usage) and
the counts of the instructions that show which hardware path it takes --
tcgen05 (UTCHMMA / UTCBAR / LDTM / STTM), TMA (UTMALDG / UTMAPF), legacy tensor
cores (HMMA), async copies (LDGSTS), programmatic dependent launch
(griddepcontrol -> ACQBULK / ... see B200_PROFILING.md), MUFU exponentials.
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2501_14808_b200", "libhygen.so")
CUOBJDUMP = "/usr/local/cuda/bin/cuobjdump"
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMAPF", "HMMA", "LDGSTS",
        "LDSM", "MUFU.EX2", "FFMA2", "FADD2", "FMUL2", "LDG", "STG", "ATOMG", "RED", "SYNCS", "ELECT",
        "ACQBULK", "PREEXIT", "CCTL", "MEMBAR", "NANOSLEEP"]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
        return out.strip().split("\n")
    except Exception:
        return names


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else None
    sass = subprocess.run([CUOBJDUMP, "-sass", SO], capture_output=True, text=True).stdout
    res = subprocess.run([CUOBJDUMP, "-res-usage", SO], capture_output=True, text=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m:
            op = m.group(1)
            kernels[cur]["_total"] += 1
            for k in KEYS:
                if op == k or op.startswith(k + "."):
                    kernels[cur][k] += 1
    usage = {}
    cur = None
    for line in res.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            cur = m.group(1)
            continue
        if cur and "REG:" in line:
            reg = re.search(r"REG:(\d+)", line)
            shared = re.search(r"SHARED:(\d+)", line)
            stack = re.search(r"STACK:(\d+)", line)
            usage[cur] = (int(reg.group(1)) if reg else None, int(shared.group(1)) if shared else None,
                          int(stack.group(1)) if stack else None)
            cur = None
    names = list(kernels)
    pretty = demangle(names)
    lines = ["# SASS census of libhygen.so (cuobjdump -sass / -res-usage, sm_100a)", "",
             "Counts of the instructions that show each kernel's hardware path.  REG = registers per "
             "thread, STACK = bytes of local stack (spills), SHARED = static shared memory (the kernels' "
             "tiles are dynamic shared memory, not in this column).", ""]
    cols = [k for k in KEYS if any(kernels[n][k] for n in names)]
    lines.append("| kernel | REG | STACK | SASS | " + " | ".join(cols) + " |")
    lines.append("|---|---|---|---|" + "---|" * len(cols))
    for n, p in zip(names, pretty):
        if "hg" not in p:
            continue
        short = re.sub(r"\(.*", "", p).replace("hg::", "")
        tmpl = re.search(r"<[^()]*>", p)
        if tmpl and "<" not in short:
            short += tmpl.group(0)
        r = usage.get(n, (None, None, None))
        lines.append(f"| `{short}` | {r[0]} | {r[2]} | {kernels[n]['_total']} | " +
                     " | ".join(str(kernels[n][k]) for k in cols) + " |")
    text = "\n".join(lines) + "\n"
    if out_path:
        open(out_path, "w").write(text)
    print(text)


if __name__ == "__main__":
    main()

"""Per-visit SASS histogram of the walk's main loop (the loop that holds the
record load), from an object file or library built here:

    python tools/sass_hist.py paper_1109_5190_b200/build/walk.o [function-regex] [visits-per-trip]

Prints the loop's instruction count by opcode, per loop trip and per record
visit, with the pipe each opcode class issues to (B300_MICROARCH.md: FFMA /
FMUL / FADD / IMAD on the fma pipe, IADD3 / LOP3 / SEL / ISETP / FSETP /
VIMNMX / PLOP3 on the alu pipe, MUFU on xu)."""
import re
import subprocess
import sys
from collections import Counter

PIPE = {"FFMA2": "fma", "FMUL2": "fma", "FADD2": "fma", "FFMA": "fma", "FMUL": "fma", "FADD": "fma", "IMAD": "fma",
        "MUFU": "xu", "F2F": "xu", "DADD": "fp64", "LDG": "lsu", "LDL": "lsu", "STL": "lsu", "LDC": "lsu"}


def loop_of(obj, fn_re):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", out)
    best = None
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        if not re.search(fn_re, name):
            continue
        ins = []
        for ln in f.splitlines():
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        for a, t in ins:
            m = re.search(r"BRA\s+.*?0x([0-9a-f]+)", t)
            if m and int(m.group(1), 16) < a:
                body = [x for x in ins if int(m.group(1), 16) <= x[0] <= a]
                if any(("256" in x[1] or "LDG.E.128" in x[1]) and "LDG" in x[1] for x in body):
                    if best is None or len(body) > len(best[1]):
                        best = (name, body)
    return best


def main():
    obj = sys.argv[1]
    fn = sys.argv[2] if len(sys.argv) > 2 else r"k_walk2ILi4ELi1ELb0ELb0"
    vpt = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    name, body = loop_of(obj, fn)
    # a warp-uniform forward branch over a block (BRA.U: the fp32 fold every
    # BH_FOLD_TRIPS trips) is the rare path: count it apart
    rare = set()
    for a, t in body:
        m = re.search(r"BRA\.U\s+.*?0x([0-9a-f]+)", t)
        if m and int(m.group(1), 16) > a:
            rare |= {x[0] for x in body if a < x[0] < int(m.group(1), 16)}
    if rare:
        print(f"(excluding {len(rare)} instructions of a warp-uniform rare block)")
    body = [x for x in body if x[0] not in rare]
    c = Counter()
    for _, t in body:
        op = t.split()[1] if t.startswith("@") else t.split()[0]
        c[op.split(".")[0]] += 1
    tot = sum(c.values())
    print(f"{name}: {tot} instructions per loop trip, {vpt} visits per trip -> {tot / vpt:.1f} per visit")
    by_pipe = Counter()
    for op, k in sorted(c.items(), key=lambda x: -x[1]):
        pipe = PIPE.get(op, "alu" if op not in ("BRA", "VOTE", "UIADD3", "UISETP", "UMOV", "CS2R") else "other")
        by_pipe[pipe] += k
        print(f"  {op:8s} {k:4d}  {k / vpt:5.1f}/visit  [{pipe}]")
    print("  by pipe per visit:", {p: round(k / vpt, 1) for p, k in by_pipe.items()})


if __name__ == "__main__":
    main()

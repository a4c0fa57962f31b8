"""Static register / spill table and SASS instruction mix of the hot kernels
(CPU only: cuobjdump on the built library).

    python tools/sass_mix.py > profiles/r02_sass_mix.txt
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1904_08684_b200", "_lib", "libqfswe.so")
# kernels the BASELINE configs launch (bench.py per_config)
HOT = {
    "C1/C2 stage (k<=2, MMS, uni table)": r"stage_kernel<(1|2), 1158>",
    "C3-C5 stage (walls, no overflow)": r"stage_kernel<(2|3|4), 144>",
    "C5 stage (walls, overflow path)": r"stage_kernel<4, 208>",
    "k=4 volume": r"volume_kernel<4, [01], false>",
    "k=4 velocity": r"velocity_kernel<4, false>",
}
GROUPS = {
    "FP64 FMA/MUL/ADD": ("DFMA", "DMUL", "DADD"),
    "FP64 other (DSETP, DMNMX, MUFU.RSQ64H)": ("DSETP", "DMNMX", "MUFU"),
    "global loads": ("LDG",),
    "global stores": ("STG",),
    "shared ld/st": ("LDS", "STS"),
    "constant loads": ("LDC", "ULDC"),
    "local (spill) ld/st": ("LDL", "STL"),
    "async copy / barrier": ("LDGSTS", "BAR", "LDGDEPBAR", "DEPBAR"),
    "integer / address": ("IMAD", "IADD3", "LEA", "SHF", "LOP3", "ISETP", "IMNMX", "SEL", "ULEA",
                          "UIADD3", "UIMAD", "USHF", "ULOP3", "UISETP", "USEL", "UMOV", "S2R",
                          "S2UR", "IABS", "POPC", "FLO", "VOTE", "VOTEU", "SHFL", "R2UR"),
    "moves / predicates": ("MOV", "PLOP3", "P2R", "R2P", "FSEL", "FSETP", "CS2R"),
    "control": ("BRA", "EXIT", "BSSY", "BSYNC", "WARPSYNC", "CALL", "RET", "NOP", "YIELD",
                "BMOV", "BREAK"),
}


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines()


def main():
    res = subprocess.run(["cuobjdump", "--dump-resource-usage", LIB], capture_output=True,
                         text=True).stdout
    usage = {}
    for m in re.finditer(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)",
                         res):
        usage[m.group(1)] = tuple(int(x) for x in m.groups()[1:])
    dem = dict(zip(usage, demangle(list(usage))))
    print("# registers / stack (spill) bytes per thread, static shared, per kernel instance")
    print("# (cuobjdump --dump-resource-usage of _lib/libqfswe.so, sm_100a)")
    for mangled, (reg, stack, shared, local) in sorted(usage.items(), key=lambda kv: dem[kv[0]]):
        name = dem[mangled].split("(")[0].replace("void ", "")
        if re.search(r"stage_kernel|volume_kernel|velocity_kernel|ghost_kernel|halo_trace", name):
            print(f"{name:45s} REG {reg:4d}  STACK {stack:5d} B  SHARED {shared:6d} B")
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if cur and m:
            funcs[cur][m.group(2).split(".")[0]] += 1
    dn = dict(zip(funcs, demangle(list(funcs))))
    print("\n# static SASS instruction mix (share of the kernel's instructions)")
    for label, pat in HOT.items():
        for mangled, cnt in sorted(funcs.items(), key=lambda kv: dn[kv[0]]):
            name = dn[mangled].split("(")[0].replace("void ", "").replace("qf::", "")
            if not re.search(pat, name):
                continue
            tot = sum(cnt.values())
            parts = []
            for g, ops in GROUPS.items():
                n = sum(cnt[o] for o in ops)
                if n:
                    parts.append(f"{g} {100.0 * n / tot:.1f}%")
            other = tot - sum(sum(cnt[o] for o in ops) for ops in GROUPS.values())
            print(f"{label} :: {name}: {tot} instructions; " + "; ".join(parts)
                  + f"; other {100.0 * other / tot:.1f}%")


if __name__ == "__main__":
    sys.exit(main())

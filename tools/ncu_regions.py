"""Aggregate an ncu source page (cuda,sass) into kernel regions (device
function / generated operator) -> share of warp instructions and stalls."""
import collections
import csv
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rep, order=2):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    ksrc = open(os.path.join(ROOT, "paper_1904_08684_b200/csrc/qf_kernels.cu")).read().splitlines()
    gsrc = open(os.path.join(ROOT, f"paper_1904_08684_b200/csrc/generated/qf_order{order}.cuh")
                ).read().splitlines()
    marks = {}  # line -> region label inside stage_kernel
    for i, l in enumerate(ksrc):
        if "if (QF_EN_VOL" in l: marks[i] = "volume"
        if "if (QF_EN_SRC" in l: marks[i] = "source"
        if "if (P.forcing)" in l: marks[i] = "forcing"
        if "if (QF_EN_EDGE" in l: marks[i] = "edge loop"
        if "SSP-RK combination" in l: marks[i] = "epilogue"
        if "// phase A: own trace" in l: marks[i] = "phase A"
        if "// phase A2: traces" in l: marks[i] = "phase A2"
        if "out-of-block neighbour requests" in l: marks[i] = "requests"
        if "stage_kernel(Tab T" in l: marks[i] = "prologue"

    def kregion(ln):
        for i in range(ln - 1, -1, -1):
            l = ksrc[i]
            if i in marks:
                return "stage:" + marks[i]
            if l.startswith("__device__ __forceinline__") or "__device__ __forceinline__ void edge_term" in l:
                return "fn:" + l.split("(")[0].split()[-1]
        return "?"

    def gregion(ln):
        for i in range(ln - 1, -1, -1):
            if "static __device__" in gsrc[i]:
                return "gen:" + gsrc[i].split("(")[0].split()[-1]
        return "gen:?"

    cur, hdr = None, None
    agg = collections.defaultdict(lambda: [0, 0])
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or r[0] == "":
            continue
        try:
            ie, ss, ln = int(r[7] or 0), int(r[4] or 0), int(r[0])
        except ValueError:
            continue
        if cur == "qf_kernels.cu":
            key = kregion(ln)
        elif cur.startswith("qf_order"):
            key = gregion(ln)
        elif cur == "qf_device.cuh":
            key = "device.cuh (scenario/forcing math)"
        else:
            key = cur
        agg[key][0] += ie
        agg[key][1] += ss
    tot = sum(v[0] for v in agg.values())
    tots = sum(v[1] for v in agg.values())
    print(f"total warp instructions {tot}, stall samples {tots}")
    for k, (ie, ss) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        if ie or ss:
            print(f"{k:45s} inst {ie / tot:6.3f}   stall-samples {ss / max(tots, 1):6.3f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 2)

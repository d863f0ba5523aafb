"""Per-phase time of the block-iteration megakernel from its trace (profiles/r01g_arn_step_phases.md).

    SKC_TRACE_ORTH=1 python tools/time_c2.py 1 2> trace.err
    python tools/phase_breakdown.py trace.err > out.md

Each `[step k=..]` line holds CTA 0's per-phase times of one block iteration; unused slots
(the last block iteration builds no next candidate) print garbage and are skipped.
"""
import collections
import re
import sys

DESC = {
    "upd": "block-MGS rounds: stream V_i, update the on-chip candidate (sstep.hpp:337-354)",
    "pass1": "conditional second orthogonalization pass (needs_reorth, sstep.hpp:356-373)",
    "cross": "cross products [V_0..V_{k-1}, cand]^T cand and W (sstep.hpp:401-414, 392-399)",
    "powers": "candidate powers A^j seed, row-streamed (sstep.hpp:330-334)",
    "Zdots": "Scalar1 products V_i^T z, z.z (sstep.hpp:305-310)",
    "seed": "seed = z - sum V_i h_i, ||seed||^2 (sstep.hpp:311-316)",
    "s1": "reduce Scalar1 partials in every CTA + k Gram solves",
    "scal": "reduce each MGS round's partials + Gram solve (per round)",
    "rsync": "grid barriers between MGS rounds",
    "r0dots": "round-0 products V_0^T cand",
    "check": "reduce cross partials, reorthogonalization test",
    "s2": "nu, invariant-subspace test, normalisation",
    "z": "z = A v (one stencil sweep)",
    "xsync": "grid barrier after the cross products",
}


def main(path):
    tot = collections.Counter()
    n = fired = 0
    for line in open(path):
        if not line.startswith("[step"):
            continue
        n += 1
        for key in ("z", "Zdots", "s1", "seed", "s2", "powers", "r0dots", "cross", "check", "pass1"):
            m = re.search(r"[ (|]%s ([0-9.]+)" % key, line)
            if m and float(m.group(1)) < 1e6:
                tot[key] += float(m.group(1))
        for a, b, c in re.findall(r"\(scal ([0-9.]+), upd ([0-9.]+), sync ([0-9.]+)\)", line):
            if float(a) < 1e6:
                tot["scal"] += float(a)
                tot["upd"] += float(b)
                tot["rsync"] += float(c)
        m = re.search(r"pass1 ([0-9.]+)", line)
        if m and float(m.group(1)) > 5:
            fired += 1
        m = re.search(r"\| znext [0-9.]+ cross [0-9.]+ sync ([0-9.]+)", line)
        if m:
            tot["xsync"] += float(m.group(1))
    total = sum(tot.values())
    print(f"{n} block iterations; the second orthogonalization pass fired in {fired} ({fired / max(1, n):.0%}).\n")
    print("| phase | us / block iteration | share | what |\n|---|---|---|---|")
    for k, v in tot.most_common():
        print(f"| {k} | {v / n:.1f} | {v / total:.3f} | {DESC[k]} |")
    print(f"| **total** | {total / n:.1f} | 1 | |")


if __name__ == "__main__":
    main(sys.argv[1])

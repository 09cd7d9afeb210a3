"""Regenerates the DESIGN.md §4.4 results table from profiles/r01_forms_table.jsonl."""
import json
import re

NAMES = {"C1": "C1 P1 mass 2D N=256 (parity cfg)", "C1b": "C1b P1 mass 2D N=4096",
         "C2": "**C2 P2 Laplace 3D N=107 Q=4 (bench)**", "C3a": "C3a P3 Helmholtz+κ 2D Q=12",
         "C3b": "C3b P3 Helmholtz+κ 3D Q=24", "C4": "C4 P2 elasticity 3D N=128", "C5-adv-P1": "C5 advection P1 Q=4",
         "C5-adv-P2": "C5 advection P2 Q=14", "C5-adv-P3": "C5 advection P3 Q=24", "C5-adv-P4": "C5 advection P4 Q=46",
         "C5-hyp-P1": "C5 hyperelastic P1 Q=4", "C5-hyp-P2": "C5 hyperelastic P2 Q=14",
         "C5-hyp-P3": "C5 hyperelastic P3 Q=24", "C5-hyp-P4": "C5 hyperelastic P4 Q=46"}
HEAD = "| config | cells | DOFs | bound | t_roof µs | step µs (zero y) | GDOF/s | roofline frac | kernel (auto schedule) |"


def short(plan):
    k = plan.split(" | ")[0]
    fz = ", fused y zeroing" if "+fused-zero" in k else ""
    k = k.replace(" +fused-zero", "")
    if k.startswith("femgpu_dmma"):
        tq = re.search(r"TQ=(\d+)", k).group(1)
        j = re.search(r"joint=(\d)", k).group(1)
        pf = re.search(r"prefetch=(\d)", k).group(1)
        b = re.search(r"basis=(\w+)", k).group(1)
        return "femgpu_dmma T^Q=%s%s%s%s%s" % (tq, ", joint 2" if j == "2" else "", ", prefetch" if pf == "1" else "",
                                               ", Φ/Ψ via L1" if b == "l1" else "", fz)
    if k.startswith("femgpu_macro"):
        return k.replace(" block=64", "").replace(" block=32", ", 32-thread CTAs") + fz
    if k.startswith("femgpu_scpt"):
        c = re.search(r"cells/thread=(\d)", k).group(1)
        m = re.search(r"minCTAs=(\d+)", k).group(1)
        return ("femgpu_scpt" + (" %s cells/thread" % c if c != "1" else "") + (" (≥%s CTAs/SM)" % m if m != "1" else "")
                + (", rolled q-loop" if "q-loop" in k else "") + fz)
    return k


def main():
    s = open("DESIGN.md").read()
    a = s.index(HEAD)
    b = s.index("7 of 14 benchmark configurations reach")
    rows = [json.loads(line) for line in open("profiles/r01_forms_table.jsonl")][1:]
    out = [HEAD, "|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        frac = r["frac_step"]
        cells = "%.2fM" % (r["cells"] / 1e6) if r["cells"] >= 1e6 else "%dk" % (r["cells"] // 1000)
        dofs = "%.2fM" % (r["dofs"] / 1e6) if r["dofs"] >= 1e6 else "%dk" % (r["dofs"] // 1000)
        fr = ("**%.2f**" if frac >= 0.5 else "%.2f") % frac
        if r["config"] == "C1":
            fr += " (launch-bound)"
        if r.get("clocks", {}).get("reasons"):
            fr += " (%s, %d MHz)" % (",".join(r["clocks"]["reasons"]), r["clocks"]["sm_mhz"])
        out.append("| %s | %s | %s | %s | %.0f | %.0f (%.0f) | %.1f | %s | %s |" % (
            NAMES[r["config"]], cells, dofs, r["bound"].upper(), r["t_roof_us"], r["step_us"], r["zero_us"], r["gdofs"],
            fr, short(r["plan"])))
    open("DESIGN.md", "w").write(s[:a] + "\n".join(out) + "\n\n" + s[b:])


if __name__ == "__main__":
    main()

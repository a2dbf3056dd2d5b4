"""Regenerate the tables of profiles/r02_scaling.md from profiles/r02_scale/*.json
and profiles/r02_bench_n1.json (development tool)."""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = lambda *a: os.path.join(ROOT, *a)


def L(n):
    return json.load(open(P("profiles", "r02_scale", f"{n}.json")))


def main():
    n1 = json.load(open(P("profiles", "r02_bench_n1.json")))["value"]
    s = open(P("profiles", "r02_scaling.md")).read()
    rows = []
    for N in (2, 4):
        for m in ("basic", "diagonal", "full"):
            d = L(f"ac_n{N}_{m}")
            h = d["halo"]
            v = f"**{d['value']:.1f}**" if m == "full" else f"{d['value']:.1f}"
            rows.append(f"| {N} | {','.join(map(str, d['config']['topology']))} | {m} | {v} | "
                        f"{d['ms_per_step']:.3f} | {100 * d['value'] / (n1 * N):.1f}% | "
                        f"{100 * h['exposed_frac']:.1f}% | {d['e2e']['value']:.1f} |")
    a = s.index("| N | topology | mode | GPts/s | ms/step | weak eff.")
    b = s.index("(4,1,1) on 4 GPUs")
    s = (s[:a] + f"| N | topology | mode | GPts/s | ms/step | weak eff. vs {n1:.1f} x N | "
         "exposed halo | e2e GPts/s |\n|---|---|---|---|---|---|---|---|\n" + "\n".join(rows) +
         "\n\n" + s[b:])
    t2, t4 = L("tti_n2_full"), L("tti_n4_full")
    s = re.sub(r"\| 2 \| 2,1,1 \| [0-9.]+ \| [0-9.]+ \| — \| ~0 \|",
               f"| 2 | 2,1,1 | {t2['value']:.1f} | {t2['ms_per_step']:.2f} | — | ~0 |", s, count=1)
    s = re.sub(r"\| 4 \| 2,2,1 \| [0-9.]+ \| [0-9.]+ \| [0-9.]+% \| ~0 \|",
               f"| 4 | 2,2,1 | {t4['value']:.1f} | {t4['ms_per_step']:.2f} | "
               f"{100 * t4['value'] / (2 * t2['value']):.1f}% | ~0 |", s, count=1)
    e1 = L("el_n1") if os.path.exists(P("profiles", "r02_scale", "el_n1.json")) else None
    e2, e4, e4f = L("el_n2_diagonal"), L("el_n4_diagonal"), L("el_n4_full")
    a = s.index("## C4: elastic")
    b = s.index("## C5:")
    n1row = (f"| 1 | 1,1,1 | — | {e1['value']:.1f} | {e1['ms_per_step']:.2f} | — |\n" if e1 else "")
    s = s[:a] + ("## C4: elastic staggered SO-8, 1024^3 global\n\n"
                 "| N | topology | mode | GPts/s | ms/step | exposed |\n|---|---|---|---|---|---|\n"
                 + n1row +
                 f"| 2 | 2,1,1 | diagonal | {e2['value']:.1f} | {e2['ms_per_step']:.2f} | "
                 f"{100 * e2['halo']['exposed_frac']:.1f}% |\n"
                 f"| 4 | 2,2,1 | diagonal | {e4['value']:.1f} | {e4['ms_per_step']:.2f} | "
                 f"{100 * e4['halo']['exposed_frac']:.1f}% |\n"
                 f"| 4 | 2,2,1 | full | {e4f['value']:.1f} | {e4f['ms_per_step']:.2f} | "
                 f"{100 * e4f['halo']['exposed_frac']:.1f}% |\n\n") + s[b:]
    v2, v4 = L("visco_n2_full"), L("visco_n4_full")
    a = s.index("## C5:")
    b = s.index("Exposed halo = (step")
    s = s[:a] + ("## C5: viscoelastic SO-16, 1024^3 global, mode full\n\n"
                 "| N | topology | GPts/s | ms/step | exposed |\n|---|---|---|---|---|\n"
                 f"| 2 | 2,1,1 | {v2['value']:.1f} | {v2['ms_per_step']:.2f} | ~0 |\n"
                 f"| 4 | 2,2,1 | {v4['value']:.1f} | {v4['ms_per_step']:.2f} | "
                 f"{100 * v4['halo']['exposed_frac']:.1f}% |\n\n") + s[b:]
    s = re.sub(r"acoustic SO-8 1024\^3: \*\*[0-9.]+ GPts/s\*\*", f"acoustic SO-8 1024^3: **{n1:.1f} GPts/s**", s)
    open(P("profiles", "r02_scaling.md"), "w").write(s)


if __name__ == "__main__":
    main()

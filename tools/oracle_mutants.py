"""Mutation check of the CPU oracle's pins.

Each mutant is one plausible slip in oracle/oracle.cpp (a dropped or halved
term, a wrong sign, index or time level, a wrong average).  It is compiled to
a scratch library and the CPU pin suites (tests/test_oracle_pins.py and
tests/test_oracle_second_coding.py; not the FLOP-count bookkeeping test) are
run against it through PF_ORACLE_LIB.  A mutant must make at least one of them
fail; the report lists the first failing test per mutant.

usage: python tools/oracle_mutants.py [--out profiles/r02_oracle_mutants.md]
"""
import argparse
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oracle.cpp")

MUTANTS = [
    ("kappa term of dc/dT: sign flipped (O5.5)",
     "dcdT = dcdT + hn[a] * (R(p.m[a][c]) - q.mu[c]", "dcdT = dcdT + hn[a] * (R(p.m[a][c]) + q.mu[c]"),
    ("kappa term of dc/dT: halved (O5.5)",
     "R(2.0 * p.A1[a][c] / (twoA * twoA))", "R(1.0 * p.A1[a][c] / (twoA * twoA))"),
    ("m term of dc/dT dropped (O5.5)",
     "dcdT = dcdT + hn[a] * (R(p.m[a][c]) - q.mu[c]", "dcdT = dcdT + hn[a] * (R(0.0) - q.mu[c]"),
    ("J_at tangential face gradient (lo+hi)/1 (O5.8, D3C19)",
     "(lo.gn[a][e] + hi.gn[a][e]) / R(2.0)", "(lo.gn[a][e] + hi.gn[a][e]) / R(1.0)"),
    ("J_at tangential face gradient (lo-hi)/2 (O5.8, D3C19)",
     "(lo.gn[a][e] + hi.gn[a][e]) / R(2.0)", "(lo.gn[a][e] - hi.gn[a][e]) / R(2.0)"),
    ("anisotropic phi face tangential gradient /1 (O4.5, D3C19)",
     "gf[a][e] = (glo[a][e] + ghi[a][e]) / R(2.0);", "gf[a][e] = (glo[a][e] + ghi[a][e]) / R(1.0);"),
    ("mobility from phi^{n+1} instead of phi^n (O5.6, reading R9)",
     "q.M[c] = q.M[c] + q.po[a] * R(", "q.M[c] = q.M[c] + q.pn[a] * R("),
    ("face d phi/dt from one side only (O5.8)",
     "const R pd = (lo.dphi[a] + hi.dphi[a]) / R(2.0) / R(p.dt);", "const R pd = (hi.dphi[a] + hi.dphi[a]) / R(2.0) / R(p.dt);"),
    ("(c^l - c^a) from one side only (O5.8)",
     "((lo.cc[LIQ][c] - lo.cc[a][c]) + (hi.cc[LIQ][c] - hi.cc[a][c])) / R(2.0)",
     "((hi.cc[LIQ][c] - hi.cc[a][c]) + (hi.cc[LIQ][c] - hi.cc[a][c])) / R(2.0)"),
    ("h_l at the face from one cell (O5.8)",
     "const R hl = pb[LIQ] * pb[LIQ] / S;", "const R hl = hi.pn[LIQ] * hi.pn[LIQ] / S;"),
    ("chi from phi^n instead of phi^{n+1} (O5.3, reading R8)",
     "chi = chi + hn[a] / R(2.0 * A_of(p, a, c, T));", "chi = chi + ho[a] / R(2.0 * A_of(p, a, c, T));"),
    ("time level t_{n+1} in T (O1)",
     "const double t = (double)g.step * p.dt;", "const double t = (double)(g.step + 1) * p.dt;"),
    ("d a/d phi_b: wrong sign of the b-update (O4.4)",
     "dadphi[b] = dadphi[b] - gq[d] * gc[a][d];", "dadphi[b] = dadphi[b] + gq[d] * gc[a][d];"),
    ("sign of Eq. (1) read as printed (+, reading R1)",
     "star[a] = ph[a] - R(p.dt / (p.tau[a] * p.eps))", "star[a] = ph[a] + R(p.dt / (p.tau[a] * p.eps))"),
    ("Lagrange mean over N-1 phases (reading R2)",
     "mean = mean / R((double)N);", "mean = mean / R((double)(N - 1));"),
    ("triple-term coefficient of d omega dropped (O4.7)",
     "s = s + R(p.gamma3[x]) * ph[b] * ph[e];", "s = s + R(0.0) * ph[b] * ph[e];"),
    ("driving force without psibar (O4.8)",
     "out[a] = R(2.0) * ph[a] / S * (ps[a] - pbar);", "out[a] = R(2.0) * ph[a] / S * (ps[a]);"),
    ("cubic anisotropy derivative factor 16 -> 8 (O4.3)",
     "R(16.0 * p.delta[a][b])", "R(8.0 * p.delta[a][b])"),
    ("anti-trapping prefactor pi eps/4 -> pi eps/2 (Eq. 4)",
     "R(M_PI * p.eps / 4.0)", "R(M_PI * p.eps / 2.0)"),
    ("anti-trapping on the liquid-side normal n_l,d (Eq. 4)",
     "* pd * dot * na[d];", "* pd * dot * nl[d];"),
    ("diffusive flux with the harmonic instead of the arithmetic mobility (reading R11)",
     "F[c] = (lo.M[c] + hi.M[c]) / R(2.0)", "F[c] = (lo.M[c] * hi.M[c]) / R(2.0)"),
    # index slips: visible only with distinct per-phase / per-pair coefficients (params/generic.json)
    ("triple coefficient of the wrong triple in d omega (O4.7)",
     "s = s + R(p.gamma3[x]) * ph[b] * ph[e];", "s = s + R(p.gamma3[a]) * ph[b] * ph[e];"),
    ("pair coefficient gamma_ab read as gamma_a,l in d omega (O4.7)",
     "if (b != a) s = s + R(16.0 / (M_PI * M_PI) * p.gamma[a][b]) * ph[b];",
     "if (b != a) s = s + R(16.0 / (M_PI * M_PI) * p.gamma[a][N - 1 - (a == N - 1)]) * ph[b];"),
    ("anisotropy strength of the solid-liquid pair for every pair (O4.3)",
     "const R ac = R(1.0) - R(p.delta[a][b]) * (R(3.0) - R(4.0) * Q4 / q4);",
     "const R ac = R(1.0) - R(p.delta[a][N - 1 - (a == N - 1)]) * (R(3.0) - R(4.0) * Q4 / q4);"),
    ("relaxation time tau of phase 0 for every phase (Eq. 1)",
     "R(p.dt / (p.tau[a] * p.eps))", "R(p.dt / (p.tau[0] * p.eps))"),
    ("mobility D of component 0 for both components (O5.6)",
     "q.po[a] * R(p.D[a][c] / (2.0 * A_of(p, a, c, T)))", "q.po[a] * R(p.D[a][0] / (2.0 * A_of(p, a, c, T)))"),
    ("A1 of component 0 in the kappa term of dc/dT (O5.5)",
     "q.mu[c] * R(2.0 * p.A1[a][c] / (twoA * twoA))", "q.mu[c] * R(2.0 * p.A1[a][0] / (twoA * twoA))"),
    ("projection threshold from rho+1 terms (O4.11)",
     "if (val(u[jdx]) - val(t) > 0.0) theta = t;", "if (val(u[jdx]) - val(t) >= 0.0) theta = t + R(1e-3);"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_oracle_mutants.md"))
    a = ap.parse_args()
    src = open(SRC).read()
    rows = []
    tmp = tempfile.mkdtemp(prefix="oracle_mut_")
    for idx, (name, old, new) in enumerate(MUTANTS):
        assert src.count(old) >= 1, f"mutant '{name}': pattern not found"
        msrc = src.replace(old, new)
        cpp = os.path.join(tmp, f"m{idx}.cpp")
        so = os.path.join(tmp, f"m{idx}.so")
        open(cpp, "w").write(msrc)
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp",
                               "-shared", "-fPIC", "-o", so, cpp])
        env = dict(os.environ, PF_ORACLE_LIB=so, OMP_NUM_THREADS="4")
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu", "-p", "no:cacheprovider",
                            "tests/test_oracle_pins.py", "tests/test_oracle_second_coding.py",
                            "--deselect", "tests/test_oracle_pins.py::test_committed_flop_counts_match_oracle"],
                           cwd=ROOT, env=env, capture_output=True, text=True)
        failed = re.findall(r"^FAILED (\S+)", r.stdout, re.M)
        caught = r.returncode != 0 and failed
        rows.append((name, bool(caught), failed[0] if failed else "(none)"))
        print(f"{'caught' if caught else 'SURVIVED'}: {name} -> {failed[0] if failed else ''}", flush=True)
    with open(a.out, "w") as f:
        f.write("# Oracle mutation check (round 2)\n\n")
        f.write("`python tools/oracle_mutants.py`: each row is one slip in `oracle/oracle.cpp`, compiled to a scratch\n"
                "library and run against the CPU pins (`tests/test_oracle_pins.py`) and the second NumPy coding\n"
                "(`tests/test_oracle_second_coding.py`), without the FLOP-count bookkeeping test. `first failing test`\n"
                "is where pytest `-x` stopped.\n\n")
        f.write("| mutant | caught | first failing test |\n|---|---|---|\n")
        for name, c, t in rows:
            f.write(f"| {name} | {'yes' if c else '**no**'} | `{t.split('::')[-1]}` |\n")
        f.write(f"\n{sum(c for _, c, _ in rows)} of {len(rows)} mutants caught.\n")
    print(f"{sum(c for _, c, _ in rows)}/{len(rows)} caught -> {a.out}")
    return 0 if all(c for _, c, _ in rows) else 1


if __name__ == "__main__":
    sys.exit(main())

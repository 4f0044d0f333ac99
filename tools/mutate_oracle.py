"""Mutation check of the oracle pins: apply each plausible mistake to
oracle/rt_oracle.c, rebuild, run the CPU pin suites, report which tests fail,
restore.  ``python tools/mutate_oracle.py [name ...]``."""
import subprocess, shutil, sys, os
os.chdir(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
src = "oracle/rt_oracle.c"
orig = open(src).read()
muts = {
 "M1 drop /s2": ("case 3: return p->init_amp / (1.0 + r2 / s2);", "case 3: return p->init_amp / (1.0 + r2);"),
 "M2 e1:=e0 (d<=2)": ("      e1 = G * (1.0 - v);", "      e1 = G * v;"),
 "M2b e1:=e0 (d=3)": ("      e1 = G * (v2 - v1);", "      e1 = G * v1;"),
 "M3 unsorted spacing": ("uint32_t lo = r1[1] < r1[2] ? r1[1] : r1[2], hi = r1[1] < r1[2] ? r1[2] : r1[1];", "uint32_t lo = r1[1], hi = r1[2];"),
 "M4 e2 wrong spacing": ("      e2 = G * (1.0 - v2);", "      e2 = G * (1.0 - v1);"),
 "M5 increment over tau": ("    h = is_leaf ? tau : S;\n    tc = tau - S;\n  }\n\n  /* Brownian", "    h = tau;\n    tc = tau - S;\n  }\n\n  /* Brownian"),
 "M6 Gamma(2) for d=3": ("double G = -log(u12 * or_unif32(r1[0]));", "double G = -log(u12);"),
}
sel = sys.argv[1:] or list(muts)
try:
    for name in sel:
        a, b = muts[name]
        assert orig.count(a) == 1, name
        open(src, "w").write(orig.replace(a, b))
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                            "tests/test_oracle_sampling.py", "tests/test_oracle_rng.py", "tests/test_oracle_pins.py"],
                           capture_output=True, text=True)
        fails = [l.split(" - ")[0] for l in r.stdout.splitlines() if l.startswith("FAILED")]
        print(f"{name}: {len(fails)} failed: {fails}", flush=True)
finally:
    open(src, "w").write(orig)
    subprocess.run([sys.executable, "-c", "import oracle; oracle.build(force=True)"])

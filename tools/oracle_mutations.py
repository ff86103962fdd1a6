"""Check that the oracle's pins can fail: apply one-line mutations of the oracle's
conventions (P1 counter layout, P8 visit-key ties, P8b step schedule) to a copy of
oracle/dpr_oracle.c, build it, run the CPU pin tests against it (DPR_ORACLE_LIB), and record
which tests failed.  Every mutation must be caught by at least one test.

    python tools/oracle_mutations.py [--out profiles/r02_oracle_mutations.json]
"""
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

SRC = os.path.join(ROOT, "oracle", "dpr_oracle.c")
TESTS = ["tests/test_oracle_rng.py", "tests/test_oracle_render.py", "tests/test_oracle_primitives.py",
         "tests/test_oracle_ring.py"]

# (name, what it breaks, old, new)
MUTATIONS = [
    ("camera_lanes_swapped", "P1 purpose 0: jx <- x1, jy <- x0",
     "jx = u01(r[0]); jy = u01(r[1]);", "jx = u01(r[1]); jy = u01(r[0]);"),
    ("camera_purpose", "P1 purpose 0 -> 1",
     "rng4(fr->seed, p, s, 0, PUR_CAMERA, 0, r);", "rng4(fr->seed, p, s, 0, PUR_LENS, 0, r);"),
    ("key_words_swapped", "P1 key = (seed hi, seed lo)",
     "uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};",
     "uint32_t key[2] = {(uint32_t)(seed >> 32), (uint32_t)(seed & 0xffffffffu)};"),
    ("counter_p_s_swapped", "P1 counter (s, p, ...)",
     "uint32_t ctr[4] = {p, s, (depth << 8) | purpose, sub};",
     "uint32_t ctr[4] = {s, p, (depth << 8) | purpose, sub};"),
    ("counter_depth_shift", "P1 counter word 2 = (depth<<4)|purpose",
     "uint32_t ctr[4] = {p, s, (depth << 8) | purpose, sub};",
     "uint32_t ctr[4] = {p, s, (depth << 4) | purpose, sub};"),
    ("ao_sub_unshifted", "P1 AO sub = k | attempt",
     "return cosine_dir(n, seed, p, s, depth, PUR_AO, (uint32_t)k << 4);",
     "return cosine_dir(n, seed, p, s, depth, PUR_AO, (uint32_t)k);"),
    ("ao_purpose", "P1 AO purpose 2 -> 3",
     "return cosine_dir(n, seed, p, s, depth, PUR_AO, (uint32_t)k << 4);",
     "return cosine_dir(n, seed, p, s, depth, PUR_BOUNCE, (uint32_t)k << 4);"),
    ("bounce_sub_offset", "P1 bounce sub = 16 + attempt",
     "return cosine_dir(n, seed, p, s, depth, PUR_BOUNCE, 0);",
     "return cosine_dir(n, seed, p, s, depth, PUR_BOUNCE, 16);"),
    ("vol_lane_rotated", "P1 volume lane (i+1)&3",
     "return u01(x[i & 3]);", "return u01(x[(i + 1) & 3]);"),
    ("vol_sub_shift", "P1 volume sub = i>>1",
     "rng4(seed, p, s, depth, purpose, subhi | (uint32_t)(i >> 2), x);",
     "rng4(seed, p, s, depth, purpose, subhi | (uint32_t)(i >> 1), x);"),
    ("vol_ao_subhi", "P1 volume AO sub = (k<<20) | i>>2",
     "v.subhi = kind == K_AO ? ((uint32_t)k << 24) : 0u;",
     "v.subhi = kind == K_AO ? ((uint32_t)k << 20) : 0u;"),
    ("vol_shadow_purpose", "P1 volume shadow purpose 5 -> 4",
     "v.purpose = kind == K_PATH ? PUR_VOL_PATH : (kind == K_SHADOW ? PUR_VOL_SHADOW : PUR_VOL_AO);",
     "v.purpose = kind == K_PATH ? PUR_VOL_PATH : (kind == K_SHADOW ? PUR_VOL_PATH : PUR_VOL_AO);"),
    ("first_candidate_tie_last", "P8 first candidate: equal t0 -> larger rank",
     "if (best < 0 || t0 < bt) { best = r; bt = t0; }",
     "if (best < 0 || t0 <= bt) { best = r; bt = t0; }"),
    ("next_candidate_tie_order", "P8 next key: equal t0 -> smaller rank after c",
     "int gt = t0 > tc || (t0 == tc && r > c);", "int gt = t0 > tc || (t0 == tc && r < c);"),
    ("next_candidate_bound_strict", "P8 next: t0 < bestT instead of t0 <= bestT",
     "if (!(t0 <= tbound)) continue;", "if (!(t0 < tbound)) continue;"),
    ("children_same_step", "P8b children traced in the resolving step",
     "ch.step = ray.step + 1;", "ch.step = ray.step;"),
    ("degenerate_not_zeroed", "R-DEGEN: zero-area triangles keep their edges",
     "if (ng.x == 0.0f && ng.y == 0.0f && ng.z == 0.0f) { *e1 = V3(0, 0, 0); *e2 = V3(0, 0, 0); }", ""),
    ("step_matrix_late", "P8b per-step S recorded in the following step",
     "L->S_step[(((batch * J->max_steps + k) * 3", "L->S_step[(((batch * J->max_steps + (k + 1 < J->max_steps ? k + 1 : k)) * 3"),
    ("forward_double_step", "P8b a forward costs two steps",
     "at = nx;\n                    ray.step++;", "at = nx;\n                    ray.step += 2;"),
]


def run(out_path):
    src = open(SRC).read()
    results = []
    with tempfile.TemporaryDirectory() as tmp:
        for name, what, old, new in MUTATIONS:
            n = src.count(old)
            if n == 0:
                raise SystemExit(f"{name}: pattern not found")
            msrc = src.replace(old, new)
            c = os.path.join(tmp, name + ".c")
            so = os.path.join(tmp, name + ".so")
            open(c, "w").write(msrc)
            subprocess.check_call(["gcc", *oracle.CFLAGS, "-o", so, c, "-lm"])
            env = dict(os.environ, DPR_ORACLE_LIB=so)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-m", "not gpu",
                                *TESTS], cwd=ROOT, env=env, capture_output=True, text=True)
            failed = sorted({ln.split(" ")[1].split(" - ")[0] for ln in r.stdout.splitlines()
                             if ln.startswith("FAILED ")})
            results.append({"mutation": name, "breaks": what, "sites": n, "caught": bool(failed),
                            "failed_tests": failed})
            print(f"{name:32s} caught={bool(failed)} ({len(failed)} tests)")
    doc = {"_what": "one-line mutations of oracle/dpr_oracle.c vs the -m 'not gpu' oracle pins "
                    "(tools/oracle_mutations.py); every mutation must be caught",
           "tests": TESTS, "all_caught": all(x["caught"] for x in results), "results": results}
    with open(out_path, "w") as f:
        json.dump(doc, f, indent=1)
    return doc


if __name__ == "__main__":
    out = os.path.join(ROOT, "profiles", "r02_oracle_mutations.json")
    for a in sys.argv[1:]:
        if a.startswith("--out="):
            out = a[6:]
    d = run(out)
    sys.exit(0 if d["all_caught"] else 1)

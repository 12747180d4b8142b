"""Runs acceptance criterion 7 (/root/reference/proj/tests/acceptance.cpp:265-298)
on the CPU oracle and prints the 128^3 reference P-bar next to the values
recorded by the reference run (/root/reference/proj/test_output.txt:48).
Writes tests/golden/c7_oracle.json. Test infrastructure only."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import oracle as O

stiff = O.neo_hookean_enu(10, 0.3)
soft = O.neo_hookean_enu(1, 0)
fbar = np.eye(3); fbar[0, 1] = 0.5
img = O.generate("sphere", (128, 128, 128), (1, 1, 1), 0.4)

def run(fac, combo, method):
    kind, cp, cnt = O.coarsen(img, fac)
    dims = tuple(128 // f for f in fac)
    nn = np.zeros((kind.size, 3))
    if combo:
        nn, fl, st = O.normals(img, fac, method=method)
    cm = O.CellMaterials(dims, kind, cp, nn, soft, stiff, combo=combo)
    t = time.time()
    r = cm.solve(fbar, scheme=1, green=1, tol=1e-7, load_steps=2, want_fields=False)
    assert r["report"]["success"], r["report"]
    return r["pbar"], r["report"], time.time() - t

out = {}
ref, rep, sec = run((1, 1, 1), False, 0)
print("ref 128^3 pbar XX %.4f XY %.4f YX %.4f YY %.4f (%.1f s, %d LS its)" % (ref[0, 0], ref[0, 1], ref[1, 0], ref[1, 1], sec, rep["ls_total"]), flush=True)
out["ref_pbar"] = ref.ravel().tolist()
out["ref_ls_total"] = rep["ls_total"]
out["recorded_reference_run"] = {"XX": 0.0007, "XY": 0.3724, "YX": 0.3667, "YY": 0.0115}
for fac in [(8, 8, 8), (16, 8, 4)]:
    errs = {}
    for name, m in (("second_moment", 1), ("barycenter", 0)):
        p, rep, sec = run(fac, True, m)
        errs[name] = float(np.linalg.norm(p - ref) / np.linalg.norm(ref))
    print("combo %s: err %.4f%% (second moment) vs %.4f%% (barycenter)" % (fac, 100 * errs["second_moment"], 100 * errs["barycenter"]), flush=True)
    out["combo_%d_%d_%d" % fac] = errs
json.dump(out, open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "c7_oracle.json"), "w"), indent=1)

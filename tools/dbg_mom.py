import os, sys, subprocess, json, numpy as np
sys.path.insert(0, ".")
import datagen as dg
if len(sys.argv) > 1:
    import paper_2208_12187_b200 as jf
    pr = dg.make_gauss2d_bounded(256, "c")
    out = {}
    for name, x in (("p0", pr.p0), ("truth", pr.truth)):
        c, g, G, bad = jf.jpass(pr.model, pr.z, x, grid=pr.grid)
        out[name] = [c, g.tolist(), G.tolist(), bad]
    print(json.dumps(out)); sys.exit(0)
res = {}
for v in ("0", "9"):
    r = subprocess.run([sys.executable, __file__, "x"], env=dict(os.environ, JF_JVARIANT=v), capture_output=True, text=True)
    res[v] = json.loads(r.stdout.strip().splitlines()[-1])
pr = dg.make_gauss2d_bounded(256, "c")
print("p0", pr.p0, "lb", pr.lb, "ub", pr.ub)
for k in ("p0", "truth"):
    c0, g0, G0, b0 = res["0"][k]; c9, g9, G9, b9 = res["9"][k]
    G0 = np.array(G0); G9 = np.array(G9); d = np.sqrt(np.diag(G9))
    print(k, "cost", c0, c9, "bad", b0, b9)
    print(" g rel", np.array2string((np.array(g0) - g9) / (d * np.sqrt(2 * c9)), precision=2))
    print(" G rel max", np.max(np.abs(G0 - G9) / np.outer(d, d)))

import os, sys, numpy as np
sys.path.insert(0, ".")
os.environ["JF_DEBUG_NOCHAIN"] = "1"
import datagen as dg
import paper_2208_12187_b200 as jf
for name, pr in (("n7", dg.make_gauss2d(96)), ("x2", dg.make_gauss2d_x2(96))):
    c, g, G, bad = jf.jpass(pr.model, pr.z, pr.p0, grid=pr.grid)
    X, Y = pr.coords()
    x = pr.p0
    def alt(sx, sy, th):
        C, S = np.cos(th), np.sin(th)
        return np.array([C*C/(2*sx*sx)+S*S/(2*sy*sy), 2*S*C*(1/(2*sy*sy)-1/(2*sx*sx)), S*S/(2*sx*sx)+C*C/(2*sy*sy)])
    cols = []
    for B in ((0, 6) if name == "x2" else (0,)):
        A, x0, y0 = x[B:B+3]
        a, b2, cc = alt(*x[B+3:B+6])
        dx, dy = X-x0, Y-y0
        E = np.exp(-(a*dx*dx + b2*dx*dy + cc*dy*dy)); AE = A*E
        cols += [E, AE*(2*a*dx+b2*dy), AE*(b2*dx+2*cc*dy), -AE*dx*dx, -AE*dx*dy, -AE*dy*dy]
    Ja = np.stack(cols + [np.ones_like(X)], 1)
    Ma = Ja.T @ Ja
    np.set_printoptions(linewidth=220, precision=2)
    d = np.sqrt(np.diag(Ma))
    print(name, "alt-space rel err\n", (G - Ma) / np.outer(d, d))

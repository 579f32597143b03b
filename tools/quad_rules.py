"""Derive the tet quadrature rules at 40 digits and
check polynomial exactness. Output literals are pasted into the product
(csrc/fem/quadrature.cpp), the C oracle and the reference harness."""
import itertools
import mpmath as mp

mp.mp.dps = 50


def exact(a, b, c):
    # integral of xi^a eta^b zeta^c over the reference tet
    return mp.factorial(a) * mp.factorial(b) * mp.factorial(c) / mp.factorial(a + b + c + 3)


def points(params):
    a1, a2, b, w1, w2, w3 = params
    pts = []
    for a, w in ((a1, w1), (a2, w2)):
        t = 1 - 3 * a
        pts += [((a, a, a), w), ((t, a, a), w), ((a, t, a), w), ((a, a, t), w)]
    t = mp.mpf(1) / 2 - b
    for p in [(b, b, t), (b, t, b), (t, b, b), (b, t, t), (t, b, t), (t, t, b)]:
        pts.append((p, w3))
    return pts


def residual(params, deg=5):
    res = []
    for a, b, c in itertools.product(range(deg + 1), repeat=3):
        if a + b + c > deg:
            continue
        s = sum(w * p[0] ** a * p[1] ** b * p[2] ** c for p, w in points(params))
        res.append(s - exact(a, b, c))
    return res


def solve14():
    x = [mp.mpf(v) for v in (0.0927352503108912, 0.3108859192633006, 0.0455037041256496,
                             0.01224884051939366, 0.01878132095300264, 0.007091003462846911)]
    for _ in range(30):
        r = residual(x)
        # least squares Newton via numerical Jacobian
        J = mp.matrix(len(r), 6)
        for k in range(6):
            h = mp.mpf(10) ** -30
            xp = list(x); xp[k] += h
            rp = residual(xp)
            for i in range(len(r)):
                J[i, k] = (rp[i] - r[i]) / h
        R = mp.matrix(r)
        dx = mp.lu_solve(J.T * J, J.T * R)
        x = [x[k] - dx[k] for k in range(6)]
    return x, max(abs(v) for v in residual(x))


if __name__ == "__main__":
    x, err = solve14()
    print("14-point degree-5 rule, max moment residual", mp.nstr(err, 5))
    for v in x:
        print(mp.nstr(v, 36))
    a = (5 - mp.sqrt(5)) / 20
    b = (5 + 3 * mp.sqrt(5)) / 20
    print("4-point a b", mp.nstr(a, 40), mp.nstr(b, 40))
    k = (1 - mp.sqrt(mp.mpf(5) / 14)) / 4
    print("Keast a", mp.nstr(k, 40), "1/2-a", mp.nstr(mp.mpf(1) / 2 - k, 40))

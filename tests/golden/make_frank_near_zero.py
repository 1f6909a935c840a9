"""High-precision truth for a Frank block whose estimate is close to 0.

Near theta = 0 the reference's Frank formulas (copula.hpp:137-172) subtract
terms of size 1/theta and 1/theta^2 (score: 1/t - g - 2 B'/B; Hessian:
-1/t^2 + g - g^2 - 2 (B''/B - (B'/B)^2)), so any fp64 evaluation of them
carries ~eps/theta^2 relative error. This script evaluates the same
pseudo-likelihood estimator in 60-digit decimal arithmetic (log c from the
closed-form Frank density, derivatives by central differences with
h = 1e-18), solves the pseudo-score equation and the SPEC variance
(O(n^2) definition), and writes the values the oracle and
the device are both compared against (tests/test_oracle.py,
tests/test_gpu_parity.py).

    python tests/golden/make_frank_near_zero.py
"""
import json
import os
from decimal import Decimal as D, getcontext

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    getcontext().prec = 60
    inp = json.load(open(os.path.join(HERE, "frank_near_zero_input.json")))
    x, y = inp["c1"], inp["c2"]
    n = len(x)

    def ranks(v):  # no ties in this block: rank = 1 + position in sorted order
        order = sorted(range(n), key=lambda i: (v[i], i))
        r = [0] * n
        for p, i in enumerate(order):
            r[i] = p + 1
        return r

    U = [D(r) / D(n + 1) for r in ranks(x)]
    V = [D(r) / D(n + 1) for r in ranks(y)]

    def logc(t, u, v):  # Frank density, theta > 0
        e = lambda z: z.exp()  # noqa: E731
        num = t * (1 - e(-t)) * e(-t * (u + v))
        den = (1 - e(-t)) - (1 - e(-t * u)) * (1 - e(-t * v))
        return (num / (den * den)).ln()

    h = D("1e-18")
    dth = lambda f, t: (f(t + h) - f(t - h)) / (2 * h)  # noqa: E731
    score = lambda t: sum(dth(lambda s: logc(s, u, v), t) for u, v in zip(U, V))  # noqa: E731
    t0, t1 = D("0.001"), D("0.0011")
    s0, s1 = score(t0), score(t1)
    for _ in range(60):  # secant to 1e-40
        t0, s0, t1 = t1, s1, t1 - s1 * (t1 - t0) / (s1 - s0)
        s1 = score(t1)
        if abs(t1 - t0) < D("1e-40"):
            break
    th = t1
    sc = [dth(lambda s: logc(s, u, v), th) for u, v in zip(U, V)]
    info = -sum((logc(th + h, u, v) - 2 * logc(th, u, v) + logc(th - h, u, v)) / (h * h) for u, v in zip(U, V)) / n

    def cross(u, v, j):
        if j == 0:
            g = lambda a: (logc(th + h, a, v) - logc(th - h, a, v)) / (2 * h)  # noqa: E731
            return (g(u + h) - g(u - h)) / (2 * h)
        g = lambda b: (logc(th + h, u, b) - logc(th - h, u, b)) / (2 * h)  # noqa: E731
        return (g(v + h) - g(v - h)) / (2 * h)

    c1 = [cross(u, v, 0) for u, v in zip(U, V)]
    c2 = [cross(u, v, 1) for u, v in zip(U, V)]
    M = D(0)
    for i in range(n):
        w1 = sum(((1 if U[i] <= U[k] else 0) - U[k]) * c1[k] for k in range(n)) / n
        w2 = sum(((1 if V[i] <= V[k] else 0) - V[k]) * c2[k] for k in range(n)) / n
        M += (sc[i] + w1 + w2) ** 2
    M /= n
    out = {"theta_hat": float(th), "sigma2": float(M / info / info / n), "digits": 60,
           "theta_hat_str": str(th)[:40], "sigma2_str": str(M / info / info / n)[:40]}
    json.dump(out, open(os.path.join(HERE, "frank_near_zero_expected.json"), "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main()

"""Drive zkl_logup_tiled_rounds directly (M61) and compare each round with a
pure-Python restatement using the device's own challenges."""
import ctypes, random, sys
sys.path[:0] = ['.']
import torch
from paper_2508_21393_b200 import _native as N, device as D
p = (1 << 61) - 1
spec = D.spec_for(p)
inv = lambda a: pow(a, p - 2, p)
random.seed(1)
n_all, tl = 10, 5
Nn, ntile = 1 << n_all, 1 << tl
r1 = n_all - tl
u = [random.randrange(p) for _ in range(n_all)]
def eqt(coords):
    t = [1]
    for c in coords:
        t = [x * v % p for x in t for v in ((1 - c) % p, c)]
    return t
table = [random.randrange(p) for _ in range(ntile)]
sec = [random.choice(table) for _ in range(Nn)]
beta = random.randrange(p)
A = [inv(s + beta) for s in sec]; S = [(s + beta) % p for s in sec]
B = [inv(t + beta) for t in table]; T = [(t + beta) % p for t in table]
M = [sec.count(t) for t in table]
al = random.randrange(p); ratio = inv(Nn // ntile)
coef = [al, -al % p, al * al % p, al ** 3 % p, -al ** 3 * ratio % p]
dev = [D.empty(spec, ntile), D.upload(A, spec), D.upload(S, spec), D.upload(B, spec), D.upload(T, spec), D.upload(M, spec)]
ptrs = (ctypes.c_void_p * 6)(*[t.data_ptr() for t in dev])
state = ctypes.create_string_buffer(bytes(64), 64)
nb = spec.nbytes
rbuf = (ctypes.c_uint8 * (r1 * 4 * nb))(); pbuf = (ctypes.c_uint8 * (r1 * nb))()
flags = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rc = N.lib().zkl_logup_tiled_rounds(spec.fid, ptrs, tl, n_all, r1, D.scalars_bytes(u, spec), D.scalars_bytes(coef, spec), flags, state, rbuf, pbuf, D.stream())
print("rc", rc, N.lib().zkl_last_error())
flat = D.decode(bytes(rbuf), spec, 4 * r1); got = [flat[4 * j:4 * j + 4] for j in range(r1)]
pt = D.decode(bytes(pbuf), spec, r1)
E = eqt(u)
full = [E, A, S, [1] * Nn, [B[i % ntile] for i in range(Nn)], [T[i % ntile] for i in range(Nn)], [M[i % ntile] for i in range(Nn)]]
def direct(tabs):
    h = len(tabs[0]) // 2
    ev = []
    for x in range(4):
        tot = 0
        for i in range(h):
            e, a, s, ind, b, tt, m = [(t[i] + x * (t[i + h] - t[i])) % p for t in tabs]
            tot += coef[0] * e * a * s + coef[1] * e * ind + coef[2] * e * b * tt + coef[3] * a + coef[4] * m * b
        ev.append(tot % p)
    return ev
def fold(t, r):
    h = len(t) // 2
    return [(t[i] + r * (t[i + h] - t[i])) % p for i in range(h)]
tabs = full
for j in range(r1):
    d = direct(tabs)
    print(j, "ok" if d == got[j] else "BAD", [(g - x) % p for g, x in zip(got[j], d)])
    tabs = [fold(t, pt[j]) for t in tabs]
Ef = D.download(dev[0], spec, ntile); Af = D.download(dev[1], spec, ntile); Sf = D.download(dev[2], spec, ntile)
print("E_out", Ef == tabs[0], "A", Af == tabs[1], "S", Sf == tabs[2])
# hypotheses for round 1
K3 = sum(B[i] * T[i] * x for i, x in enumerate(eqt(u[r1:]))) % p
SMB = sum(M[i] * B[i] for i in range(ntile)) % p
el = eqt(u[r1:])
def formula(j, Aj, Sj, C, ehcoords=None, uj=None, Pmode=0):
    h = len(Aj) // 2
    K = h >> tl
    eh = eqt(u[j + 1:r1] if ehcoords is None else ehcoords)
    P = [0, 0, 0]; sa0 = sad = 0
    for i in range(h):
        k, ti = i >> tl, i & (ntile - 1)
        w = eh[k] * el[ti] % p
        a0, a1, s0, s1 = Aj[i], Aj[i + h], Sj[i], Sj[i + h]
        ad, sd = (a1 - a0) % p, (s1 - s0) % p
        P[0] += w * a0 * s0; P[1] += w * a1 * s1; P[2] += w * ad * sd
        sa0 += a0; sad += ad
    P = [x % p for x in P]
    q = [P[0], P[1], (2 * P[1] + 2 * P[2] - P[0]) % p, (3 * P[1] + 6 * P[2] - 2 * P[0]) % p]
    uu = u[j] if uj is None else uj
    return [(C * ((1 - uu) + x * (2 * uu - 1)) * (coef[0] * q[x] + coef[1] + coef[2] * K3) + coef[3] * (sa0 + x * sad) + coef[4] * K * SMB) % p for x in range(4)]
A1, S1 = fold(A, pt[0]), fold(S, pt[0])
C1 = ((1 - u[0]) + pt[0] * (2 * u[0] - 1)) % p
print("H0 correct", formula(1, A1, S1, C1) == direct([fold(t, pt[0]) for t in full]))
print("H1 C=1", formula(1, A1, S1, 1) == got[1])
print("H2 u0", formula(1, A1, S1, C1, uj=u[0]) == got[1])
print("H3 eh round0 table prefix", formula(1, A1, S1, C1, ehcoords=u[1:r1 - 1]) == got[1])
print("H4 C=r", formula(1, A1, S1, pt[0]) == got[1])

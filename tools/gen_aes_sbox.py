"""Generate csrc/aes_sbox_bs.cuh: a bitsliced (straight-line XOR/AND) circuit
for the AES S-box, verified on all 256 inputs before anything is written.
The emitted circuit is Boyar-Peralta's depth-16 SLP (128 gates); a circuit
derived here via the tower field GF((2^4)^2) (168 gates) is verified too, as
an independent check of the reference S-box and the simulator.  Product-side code generator: it does
NOT use oracle/ (the S-box reference here is computed independently from the
FIPS-197 5.1.1 definition).

Circuit: S(x) = A . inv(x) + 0x63, inv via an isomorphism phi: GF(2^8)_AES ->
GF(2^4)[z]/(z^2 + z + lam) with GF(2^4) = GF(2)[w]/(w^4 + w + 1):
  g = a z + b,  Delta = lam a^2 + a b + b^2,  g^-1 = (a Delta^-1) z + (a + b) Delta^-1
Linear maps (phi, A.phi^-1) are emitted as XOR networks with greedy common-pair
elimination (Paar); GF(2^4) multiplications as schoolbook AND/XOR; the 4-bit
inverse from its algebraic normal form.
    python tools/gen_aes_sbox.py
"""
import itertools
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "paper_2301_10904_b200", "csrc", "aes_sbox_bs.cuh")


# ---------------------------------------------------------------- reference S-box (FIPS-197 5.1.1)
def gmul(a, b, poly=0x11B, bits=8):
    p = 0
    while b:
        if b & 1:
            p ^= a
        b >>= 1
        a <<= 1
        if a >> bits:
            a ^= poly
    return p


def sbox_ref(x):
    inv = 0 if x == 0 else next(y for y in range(1, 256) if gmul(x, y) == 1)
    out = 0
    for i in range(8):
        bit = ((inv >> i) ^ (inv >> ((i + 4) % 8)) ^ (inv >> ((i + 5) % 8)) ^ (inv >> ((i + 6) % 8)) ^
               (inv >> ((i + 7) % 8)) ^ (0x63 >> i)) & 1
        out |= bit << i
    return out


SBOX = [sbox_ref(x) for x in range(256)]
assert SBOX[0] == 0x63 and SBOX[0x53] == 0xED and SBOX[0xFF] == 0x16


# ---------------------------------------------------------------- tower field arithmetic (integers)
def g16_mul(a, b):
    return gmul(a, b, poly=0b10011, bits=4)  # w^4 + w + 1


def tower_mul(x, y, lam):  # x = (a, b) meaning a z + b
    a, b = x
    c, d = y
    ac = g16_mul(a, c)
    return (ac ^ g16_mul(a, d) ^ g16_mul(b, c), g16_mul(ac, lam) ^ g16_mul(b, d))


def find_lam():
    for lam in range(1, 16):  # z^2 + z + lam irreducible over GF(16)
        if all(g16_mul(z, z) ^ z ^ lam for z in range(16)):
            return lam
    raise AssertionError


LAM = find_lam()


def tower_pow(x, e):
    r = (0, 1)
    for _ in range(e):
        r = tower_mul(r, x, LAM)
    return r


def to_int(t):
    return (t[0] << 4) | t[1]


def find_phi():
    """Root beta of the AES polynomial in the tower field; phi(x^i) = beta^i."""
    aes_poly = [1, 1, 0, 1, 1, 0, 0, 0, 1]  # x^8 + x^4 + x^3 + x + 1, coeff of x^i
    for cand in range(2, 256):
        beta = (cand >> 4, cand & 15)
        acc = (0, 0)
        for i, c in enumerate(aes_poly):
            if c:
                p = tower_pow(beta, i)
                acc = (acc[0] ^ p[0], acc[1] ^ p[1])
        if acc == (0, 0):
            cols = [to_int(tower_pow(beta, i)) for i in range(8)]  # image of basis x^i
            # must be invertible
            if rank(cols) == 8:
                return cols
    raise AssertionError


def rank(cols):
    rows = list(cols)
    r = 0
    for bit in range(8):
        piv = next((i for i in range(r, len(rows)) if rows[i] >> bit & 1), None)
        if piv is None:
            continue
        rows[r], rows[piv] = rows[piv], rows[r]
        for i in range(len(rows)):
            if i != r and rows[i] >> bit & 1:
                rows[i] ^= rows[r]
        r += 1
    return r


PHI_COLS = find_phi()


def phi(x):
    out = 0
    for i in range(8):
        if x >> i & 1:
            out ^= PHI_COLS[i]
    return out


PHI_INV = {phi(x): x for x in range(256)}
assert len(PHI_INV) == 256


# ---------------------------------------------------------------- circuit builder
class Circuit:
    def __init__(self):
        self.ops = []  # (dst, op, a, b)
        self.n = 0

    def new(self, op, a, b):
        name = "t%d" % self.n
        self.n += 1
        self.ops.append((name, op, a, b))
        return name

    def xor(self, a, b):
        return self.new("^", a, b)

    def and_(self, a, b):
        return self.new("&", a, b)

    def xor_many(self, xs):
        xs = list(xs)
        assert xs
        acc = xs[0]
        for x in xs[1:]:
            acc = self.xor(acc, x)
        return acc

    def linear(self, inputs, rows):
        """outputs[k] = XOR of inputs[j] for j in rows[k] (sets), greedy pair sharing (Paar)."""
        rows = [set(r) for r in rows]
        sigs = list(inputs)
        while True:
            counts = {}
            for r in rows:
                for p in itertools.combinations(sorted(r), 2):
                    counts[p] = counts.get(p, 0) + 1
            if not counts:
                break
            (i, j), c = max(counts.items(), key=lambda kv: (kv[1], -kv[0][0], -kv[0][1]))
            if c < 2:
                break
            new = len(sigs)
            sigs.append(self.xor(sigs[i], sigs[j]))
            for r in rows:
                if i in r and j in r:
                    r.discard(i)
                    r.discard(j)
                    r.add(new)
        outs = []
        for r in rows:
            outs.append(self.xor_many([sigs[k] for k in sorted(r)]) if r else None)
        return outs

    def g16_mul(self, a, b):
        """a, b: 4 signals (coeff of w^0..w^3) -> product mod w^4 + w + 1."""
        c = [[] for _ in range(7)]
        for i in range(4):
            for j in range(4):
                c[i + j].append(self.and_(a[i], b[j]))
        cs = [self.xor_many(x) for x in c]
        # w^4 = w + 1, w^5 = w^2 + w, w^6 = w^3 + w^2
        return [self.xor_many([cs[0], cs[4]]), self.xor_many([cs[1], cs[4], cs[5]]),
                self.xor_many([cs[2], cs[5], cs[6]]), self.xor_many([cs[3], cs[6]])]

    def g16_const_linear(self, a, fn):
        """Any GF(2)-linear map on GF(16) given as an integer function."""
        rows = []
        for k in range(4):
            rows.append({i for i in range(4) if fn(1 << i) >> k & 1})
        return self.linear(a, rows)

    def g16_inv(self, a):
        """4-bit inverse (0 -> 0) from its algebraic normal form."""
        inv = [0] + [next(y for y in range(1, 16) if g16_mul(x, y) == 1) for x in range(1, 16)]
        monos = {}

        def mono(mask):
            if mask in monos:
                return monos[mask]
            bits = [i for i in range(4) if mask >> i & 1]
            if len(bits) == 1:
                s = a[bits[0]]
            else:
                s = self.and_(mono(mask & ~(1 << bits[-1])), a[bits[-1]])
            monos[mask] = s
            return s

        outs = []
        for k in range(4):
            f = [inv[x] >> k & 1 for x in range(16)]
            anf = f[:]  # Moebius transform
            for i in range(4):
                for x in range(16):
                    if x >> i & 1:
                        anf[x] ^= anf[x ^ (1 << i)]
            assert anf[0] == 0
            terms = [mono(m) for m in range(1, 16) if anf[m]]
            outs.append(self.xor_many(terms))
        return outs


def build():
    C = Circuit()
    x = ["x[%d]" % i for i in range(8)]  # x[i] = plane of bit i
    # input map phi: tower bits (b0..b3 = low nibble = const coeff b, a0..a3 = z coeff a)
    rows = [{i for i in range(8) if PHI_COLS[i] >> k & 1} for k in range(8)]
    y = C.linear(x, rows)
    b, a = y[0:4], y[4:8]
    # Delta = lam a^2 + a b + b^2
    a2l = C.g16_const_linear(a, lambda v: g16_mul(g16_mul(v, v), LAM))
    b2 = C.g16_const_linear(b, lambda v: g16_mul(v, v))
    ab = C.g16_mul(a, b)
    delta = [C.xor_many([a2l[k], ab[k], b2[k]]) for k in range(4)]
    dinv = C.g16_inv(delta)
    hi = C.g16_mul(a, dinv)
    apb = [C.xor(a[k], b[k]) for k in range(4)]
    lo = C.g16_mul(apb, dinv)
    t = lo + hi  # tower element bits: low nibble = const coeff, high = z coeff
    # output: A . phi^-1 (t) + 0x63
    def out_lin(v):
        inv = PHI_INV[v]
        o = 0
        for i in range(8):
            bit = ((inv >> i) ^ (inv >> ((i + 4) % 8)) ^ (inv >> ((i + 5) % 8)) ^ (inv >> ((i + 6) % 8)) ^
                   (inv >> ((i + 7) % 8))) & 1
            o |= bit << i
        return o
    rows = [{i for i in range(8) if out_lin(1 << i) >> k & 1} for k in range(8)]
    outs = C.linear(t, rows)
    return C, outs


# Boyar & Peralta, "A depth-16 circuit for the AES S-box" (2012): 128 gates
# (34 AND, 94 XOR/XNOR).  U0 = most significant input bit, S0 = most
# significant output bit, "#" = XNOR.  Verified below like the tower circuit.
BP = """
T1 = U0 + U3
T2 = U0 + U5
T3 = U0 + U6
T4 = U3 + U5
T5 = U4 + U6
T6 = T1 + T5
T7 = U1 + U2
T8 = U7 + T6
T9 = U7 + T7
T10 = T6 + T7
T11 = U1 + U5
T12 = U2 + U5
T13 = T3 + T4
T14 = T6 + T11
T15 = T5 + T11
T16 = T5 + T12
T17 = T9 + T16
T18 = U3 + U7
T19 = T7 + T18
T20 = T1 + T19
T21 = U6 + U7
T22 = T7 + T21
T23 = T2 + T22
T24 = T2 + T10
T25 = T20 + T17
T26 = T3 + T16
T27 = T1 + T12
M1 = T13 x T6
M2 = T23 x T8
M3 = T14 + M1
M4 = T19 x U7
M5 = M4 + M1
M6 = T3 x T16
M7 = T22 x T9
M8 = T26 + M6
M9 = T20 x T17
M10 = M9 + M6
M11 = T1 x T15
M12 = T4 x T27
M13 = M12 + M11
M14 = T2 x T10
M15 = M14 + M11
M16 = M3 + M2
M17 = M5 + T24
M18 = M8 + M7
M19 = M10 + M15
M20 = M16 + M13
M21 = M17 + M15
M22 = M18 + M13
M23 = M19 + T25
M24 = M22 + M23
M25 = M22 x M20
M26 = M21 + M25
M27 = M20 + M21
M28 = M23 + M25
M29 = M28 x M27
M30 = M26 x M24
M31 = M20 x M23
M32 = M27 x M31
M33 = M27 + M25
M34 = M21 x M22
M35 = M24 x M34
M36 = M24 + M25
M37 = M21 + M29
M38 = M32 + M33
M39 = M23 + M30
M40 = M35 + M36
M41 = M38 + M40
M42 = M37 + M39
M43 = M37 + M38
M44 = M39 + M40
M45 = M42 + M41
M46 = M44 x T6
M47 = M40 x T8
M48 = M39 x U7
M49 = M43 x T16
M50 = M38 x T9
M51 = M37 x T17
M52 = M42 x T15
M53 = M45 x T27
M54 = M41 x T10
M55 = M44 x T13
M56 = M40 x T23
M57 = M39 x T19
M58 = M43 x T3
M59 = M38 x T22
M60 = M37 x T20
M61 = M42 x T1
M62 = M45 x T4
M63 = M41 x T2
L0 = M61 + M62
L1 = M50 + M56
L2 = M46 + M48
L3 = M47 + M55
L4 = M54 + M58
L5 = M49 + M61
L6 = M62 + L5
L7 = M46 + L3
L8 = M51 + M59
L9 = M52 + M53
L10 = M53 + L4
L11 = M60 + L2
L12 = M48 + M51
L13 = M50 + L0
L14 = M52 + M61
L15 = M55 + L1
L16 = M56 + L0
L17 = M57 + L1
L18 = M58 + L8
L19 = M63 + L4
L20 = L0 + L1
L21 = L1 + L7
L22 = L3 + L12
L23 = L18 + L2
L24 = L15 + L9
L25 = L6 + L10
L26 = L7 + L9
L27 = L8 + L10
L28 = L11 + L14
L29 = L11 + L17
S0 = L6 + L24
S1 = L16 # L26
S2 = L19 # L28
S3 = L6 + L21
S4 = L20 + L22
S5 = L25 + L29
S6 = L13 # L27
S7 = L6 # L23
"""


def bp_circuit():
    C = Circuit()
    env = {"U%d" % i: "x[%d]" % (7 - i) for i in range(8)}
    nots = {}
    for line in BP.strip().splitlines():
        d, _, a, op, b = line.split()
        if op == "+":
            env[d] = C.xor(env[a], env[b])
        elif op == "x":
            env[d] = C.and_(env[a], env[b])
        else:  # XNOR: complement folded into the output
            env[d] = C.xor(env[a], env[b])
            nots[d] = True
    outs = [env["S%d" % (7 - k)] for k in range(8)]
    inv = [bool(nots.get("S%d" % (7 - k))) for k in range(8)]
    return C, outs, inv


def simulate(C, outs, xval):
    env = {"x[%d]" % i: (xval >> i) & 1 for i in range(8)}
    for dst, op, a, b in C.ops:
        env[dst] = env[a] ^ env[b] if op == "^" else env[a] & env[b]
    v = 0
    for k, o in enumerate(outs):
        v |= env[o] << k
    return v ^ 0x63


def simulate_bp(C, outs, inv, xval):
    v = simulate(C, outs, xval) ^ 0x63  # raw circuit value
    for k in range(8):
        if inv[k]:
            v ^= 1 << k
    return v


def main():
    C, outs = build()  # tower-field circuit: derived here, used as a cross-check
    for xv in range(256):
        assert simulate(C, outs, xv) == SBOX[xv], xv
    C, outs, inv = bp_circuit()  # emitted: fewer gates
    for xv in range(256):
        assert simulate_bp(C, outs, inv, xv) == SBOX[xv], xv
    n_and = sum(1 for o in C.ops if o[1] == "&")
    n_xor = len(C.ops) - n_and
    lines = [
        "// aes_sbox_bs.cuh -- GENERATED by tools/gen_aes_sbox.py; do not edit.",
        "// Bitsliced AES S-box (FIPS-197 5.1.1): the Boyar-Peralta depth-16 circuit, %d XOR/XNOR + %d AND" %
        (n_xor, n_and),
        "// gates, verified on all 256 inputs by the generator (which also derives and verifies a",
        "// tower-field GF((2^4)^2) circuit as an independent cross-check).  x[i] holds bit i of every",
        "// byte lane (one lane per bit of the 32-bit word); the result replaces x.",
        "#pragma once",
        "#include <cstdint>",
        "namespace dpfpir {",
        "namespace dev {",
        "__device__ __forceinline__ void aes_sbox_bs(uint32_t (&x)[8]) {",
    ]
    for dst, op, a, b in C.ops:
        lines.append("  const uint32_t %s = %s %s %s;" % (dst, a, op, b))
    for k, o in enumerate(outs):
        lines.append("  const uint32_t o%d = %s%s;" % (k, "~" if inv[k] else "", o))
    lines.append("  " + " ".join("x[%d] = o%d;" % (k, k) for k in range(8)))
    lines += ["}", "}  // namespace dev", "}  // namespace dpfpir", ""]
    with open(OUT, "w") as f:
        f.write("\n".join(lines))
    print("wrote %s: %d XOR + %d AND" % (OUT, n_xor, n_and))


if __name__ == "__main__":
    main()

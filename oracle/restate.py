"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's µGraph
evaluation path (numpy), used as a checker by tests/ and never by the product.

Parity status: PINNED against the compiled reference itself
(``oracle/_ref/libtpo_ref.so``, built from /root/reference by
``oracle/Makefile``): tests/test_oracle.py compares this restatement with the
reference on the committed golden vectors in tests/golden/ and, when the
reference library is present, on freshly generated cases.

Each function cites the reference code it restates:

* ``Rng``              — proj/core/include/tpo/util/rng.hpp:25-63 (splitmix64,
                         derive, rejection-sampled uniform, Box–Muller normal)
* ``Field``            — proj/core/src/field.cpp:43-142 (tables, add/sub/mul/div/
                         exp/sqrt, sample, sample_omega)
* ``sample_inputs`` / ``silu_tables`` — proj/core/src/ffeval.cpp:20-40
* ``Evaluator``        — proj/core/include/tpo/internal/eval_core.hpp:74-377
* ``random_test_equivalence`` — proj/core/src/equiv.cpp:34-94
* ``float_stability_filter``  — proj/core/src/stability.cpp:25-50
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence

import numpy as np

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
PHI = -1


# ---------------------------------------------------------------------------
# RNG (rng.hpp:25-63)
# ---------------------------------------------------------------------------

def _fin_np(z: np.ndarray) -> np.ndarray:
    """splitmix64 output finalizer (rng.hpp:38-40) on a uint64 array."""
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


class Rng:
    """splitmix64 stream (rng.hpp:25-63)."""

    def __init__(self, seed: int):
        self.state = seed & M64

    @staticmethod
    def derive(seed: int, stream: int) -> "Rng":
        r = Rng(seed ^ ((GAMMA * (stream + 1)) & M64))  # rng.hpp:30-34
        r.next()
        return r

    def next(self) -> int:
        self.state = (self.state + GAMMA) & M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def next_block(self, n: int) -> np.ndarray:
        """n consecutive draws in closed form: draw j = fin(state + (j+1)·γ)."""
        with np.errstate(over="ignore"):
            idx = np.arange(1, n + 1, dtype=np.uint64)
            z = np.uint64(self.state) + idx * np.uint64(GAMMA)
        self.state = (self.state + n * GAMMA) & M64
        return _fin_np(z)

    def uniform(self, n: int) -> int:
        thr = ((1 << 64) - n) % n  # rng.hpp:44-50
        while True:
            r = self.next()
            if r >= thr:
                return r % n

    def uniform_pairs(self, count: int, n1: int, n2: int):
        """`count` alternating draws uniform(n1), uniform(n2) (sample() per element,
        field.cpp:133-138), vectorised with an exact sequential fallback when a
        rejection (probability ~1e-17 per draw) occurs."""
        t1, t2 = ((1 << 64) - n1) % n1, ((1 << 64) - n2) % n2
        save = self.state
        raw = self.next_block(2 * count)
        a, b = raw[0::2], raw[1::2]
        if count and (np.any(a < np.uint64(t1)) or np.any(b < np.uint64(t2))):
            self.state = save
            xs = np.zeros(count, np.int64)
            ys = np.zeros(count, np.int64)
            for i in range(count):
                xs[i] = self.uniform(n1)
                ys[i] = self.uniform(n2)
            return xs, ys
        return (a % np.uint64(n1)).astype(np.int64), (b % np.uint64(n2)).astype(np.int64)

    def uniform_many(self, count: int, n: int) -> np.ndarray:
        t = ((1 << 64) - n) % n
        save = self.state
        raw = self.next_block(count)
        if count and np.any(raw < np.uint64(t)):
            self.state = save
            return np.array([self.uniform(n) for _ in range(count)], np.int64)
        return (raw % np.uint64(n)).astype(np.int64)

    def uniform_real(self) -> float:
        return float(self.next() >> 11) * (1.0 / 9007199254740992.0)

    def normal(self) -> float:
        u1 = self.uniform_real()
        u2 = self.uniform_real()
        if u1 < 1e-300:
            u1 = 1e-300
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586 * u2)


# ---------------------------------------------------------------------------
# Finite field Z_p x Z_q (field.hpp / field.cpp)
# ---------------------------------------------------------------------------

class ResampleNeeded(Exception):
    """field.hpp:29-31"""

    def __init__(self, code: str):
        super().__init__(code)
        self.code = code


class PoisonedExponent(Exception):
    """ErrCode::PoisonedExponent thrown as tpo::Error (field.cpp:105-108)."""


def _is_prime(n: int) -> bool:
    return n >= 2 and all(n % d for d in range(2, int(n ** 0.5) + 1))


class Field:
    """FieldParams (field.cpp:43-67).  Values are (xp, xq, qd) numpy triples."""

    def __init__(self, p: int = 227, q: int = 113, wbase: int = 4):
        if not (_is_prime(p) and _is_prime(q)):
            raise ValueError("ConfigError: p and q must be prime")
        if (p - 1) % q:
            raise ValueError("ConfigError: q must divide p-1")
        if wbase % p in (0, 1) or pow(wbase, q, p) != 1:
            raise ValueError("ConfigError: omega base must have order q")
        self.p, self.q, self.wbase = p, q, wbase
        self.inv_p = np.array([0] + [pow(x, p - 2, p) for x in range(1, p)], np.int64)
        self.inv_q = np.array([0] + [pow(x, q - 2, q) for x in range(1, q)], np.int64)
        self.sqrt_p = np.full(p, -1, np.int64)
        for r in range(p - 1, -1, -1):  # smaller root wins (field.cpp:61-66)
            self.sqrt_p[r * r % p] = r
        self.sqrt_q = np.full(q, -1, np.int64)
        for r in range(q - 1, -1, -1):
            self.sqrt_q[r * r % q] = r
        self.pow_table = None

    # elementwise ops on (xp, xq, qd) triples of equal (broadcast) shape
    def add(self, a, b):
        qd = a[2] & b[2]
        return (a[0] + b[0]) % self.p, np.where(qd, (a[1] + b[1]) % self.q, 0), qd

    def sub(self, a, b):
        qd = a[2] & b[2]
        return (a[0] + self.p - b[0]) % self.p, np.where(qd, (a[1] + self.q - b[1]) % self.q, 0), qd

    def mul(self, a, b):
        qd = a[2] & b[2]
        return a[0] * b[0] % self.p, np.where(qd, a[1] * b[1] % self.q, 0), qd

    def div(self, a, b):
        if np.any(b[0] == 0):
            raise ResampleNeeded("DivByZero")
        qd = a[2] & b[2]
        if np.any(qd & (b[1] == 0)):
            raise ResampleNeeded("DivByZero")
        return (a[0] * self.inv_p[b[0]] % self.p, np.where(qd, a[1] * self.inv_q[b[1]] % self.q, 0),
                qd)

    def exp(self, a, omega: int):
        if not np.all(a[2]):
            raise PoisonedExponent("exponent depends on a prior exponentiation")
        tab = np.array([pow(omega, e, self.p) for e in range(self.q)], np.int64)
        xp = tab[a[1]]
        return xp, np.zeros_like(xp), np.zeros(np.shape(xp), bool)

    def sqrt(self, a):
        rp = self.sqrt_p[a[0]]
        if np.any(rp < 0):
            raise ResampleNeeded("NonResidue")
        rq = np.where(a[2], self.sqrt_q[a[1]], 0)
        if np.any(rq < 0):
            raise ResampleNeeded("NonResidue")
        return rp, rq, a[2].copy()

    def sample_omega(self, rng: Rng) -> int:
        return pow(self.wbase, rng.uniform(self.q), self.p)  # field.cpp:140-142


class FFSem:
    """FFSemantics (ffeval.hpp:35-56).  Tensor values are (xp, xq, qd) arrays."""

    kind = "ff"

    def __init__(self, field: Field, omega: int, silu=None):
        self.f, self.omega, self.silu_t = field, omega, silu

    def zeros(self, shape):
        return (np.zeros(shape, np.int64), np.zeros(shape, np.int64), np.ones(shape, bool))

    add = property(lambda s: s.f.add)
    mul = property(lambda s: s.f.mul)
    div = property(lambda s: s.f.div)

    def exp(self, a):
        return self.f.exp(a, self.omega)

    def sqrt(self, a):
        return self.f.sqrt(a)

    def silu(self, a):
        if self.silu_t is None:
            raise RuntimeError("Unsupported: silu tables not sampled")
        tp, tq = self.silu_t
        return tp[a[0]], np.where(a[2], tq[a[1]], 0), a[2].copy()

    # structural helpers
    @staticmethod
    def take(a, idx):
        return tuple(x.reshape(-1)[idx] for x in a)

    @staticmethod
    def shape(a):
        return a[0].shape

    @staticmethod
    def reshape(a, s):
        return tuple(x.reshape(s) for x in a)

    def matmul(self, a, b):
        """eval_core.hpp:181-203: acc = zero; acc = add(acc, mul(a,b)) — order-free in Z_p."""
        p, q = self.f.p, self.f.q
        xp = np.matmul(a[0], b[0]) % p
        qd_a = np.all(a[2], axis=-1, keepdims=True)  # structural per row/col
        qd_b = np.all(b[2], axis=-2, keepdims=True)
        qd = np.broadcast_to(qd_a & qd_b, xp.shape).copy()
        # elementwise poison: an output is q-defined iff every product term is
        qd_full = np.matmul(a[2].astype(np.int64), b[2].astype(np.int64)) == a[0].shape[-1]
        qd = qd & qd_full
        xq = np.where(qd, np.matmul(np.where(a[2], a[1], 0), np.where(b[2], b[1], 0)) % q, 0)
        return xp, xq, qd

    def grouped_sum(self, a, dim, group):
        shp = list(a[0].shape)
        new = shp[:dim] + [shp[dim] // group, group] + shp[dim + 1:]
        xp = a[0].reshape(new).sum(axis=dim + 1) % self.f.p
        qd = np.all(a[2].reshape(new), axis=dim + 1)
        xq = np.where(qd, a[1].reshape(new).sum(axis=dim + 1) % self.f.q, 0)
        return xp, xq, qd

    @staticmethod
    def broadcast(a, shape):
        return tuple(np.broadcast_to(x, shape).copy() for x in a)

    @staticmethod
    def copy(a):
        return tuple(x.copy() for x in a)

    @staticmethod
    def setitem(dst, sl, val):
        for d, v in zip(dst, val):
            d[sl] = v

    @staticmethod
    def getitem(a, sl):
        return tuple(x[sl] for x in a)


class FloatSem:
    """FloatSemantics<double> (interp.hpp:27-38).  numpy matmul reassociates the
    sums; differences vs the reference are at the 1e-15 relative level."""

    kind = "float"

    def __init__(self, dtype=np.float64):
        self.dtype = dtype

    def zeros(self, shape):
        return np.zeros(shape, self.dtype)

    @staticmethod
    def add(a, b):
        return a + b

    @staticmethod
    def mul(a, b):
        return a * b

    @staticmethod
    def div(a, b):
        with np.errstate(divide="ignore", invalid="ignore"):
            return a / b

    @staticmethod
    def exp(a):
        with np.errstate(over="ignore"):
            return np.exp(a)

    @staticmethod
    def sqrt(a):
        with np.errstate(invalid="ignore"):
            return np.sqrt(a)

    @staticmethod
    def silu(a):
        with np.errstate(over="ignore"):
            return a / (1.0 + np.exp(-a))

    @staticmethod
    def take(a, idx):
        return a.reshape(-1)[idx]

    @staticmethod
    def shape(a):
        return a.shape

    @staticmethod
    def reshape(a, s):
        return a.reshape(s)

    @staticmethod
    def matmul(a, b):
        return np.matmul(a, b)

    @staticmethod
    def grouped_sum(a, dim, group):
        shp = list(a.shape)
        return a.reshape(shp[:dim] + [shp[dim] // group, group] + shp[dim + 1:]).sum(axis=dim + 1)

    @staticmethod
    def broadcast(a, shape):
        return np.broadcast_to(a, shape).copy()

    @staticmethod
    def copy(a):
        return a.copy()

    @staticmethod
    def setitem(dst, sl, val):
        dst[sl] = val

    @staticmethod
    def getitem(a, sl):
        return a[sl]


# ---------------------------------------------------------------------------
# Evaluator (eval_core.hpp:74-377)
# ---------------------------------------------------------------------------

def _dm(j, grid_axes=True):
    out = []
    for k in (("x", "y", "z") if grid_axes else ("i",)):
        if k not in j:
            break
        out.append(PHI if j[k] == "phi" else int(j[k]))
    return out


def _bshape(a, b):
    r = max(len(a), len(b))
    a = (1,) * (r - len(a)) + tuple(a)
    b = (1,) * (r - len(b)) + tuple(b)
    return tuple(max(x, y) for x, y in zip(a, b))


class Evaluator:
    def __init__(self, sem):
        self.s = sem

    def run(self, g: dict, inputs: Sequence):
        """eval_core.hpp:81-104 — ops in list order."""
        s = self.s
        vals = [None] * len(g["tensors"])
        if len(inputs) != len(g["inputs"]):
            raise ValueError("ShapeMismatch: input count")
        for t, x in zip(g["inputs"], inputs):
            if tuple(s.shape(x)) != tuple(g["tensors"][t]["shape"]):
                raise ValueError("ShapeMismatch: input tensor shape")
            vals[t] = x
        for op in g["ops"]:
            if op["type"] == "graphdef":
                self._graphdef(g, op, vals)
                continue
            ins = [vals[t] for t in op["inputs"]]
            vals[op["outputs"][0]] = self._predef(op, ins, g["tensors"][op["outputs"][0]]["shape"])
        return [vals[t] for t in g["outputs"]]

    def _predef(self, op, ins, out_shape):
        """eval_core.hpp:109-158"""
        s, t = self.s, op["type"]
        if t == "matmul":
            return s.matmul(ins[0], ins[1])
        if t == "concatmatmul":
            return s.add(s.matmul(ins[0], ins[2]), s.matmul(ins[1], ins[3]))
        if t == "sum":
            return s.grouped_sum(ins[0], op["attrs"]["dim"], op["attrs"]["group"])
        if t in ("ewadd", "ewmul", "ewdiv"):
            shp = _bshape(s.shape(ins[0]), s.shape(ins[1]))
            a, b = s.broadcast(ins[0], shp), s.broadcast(ins[1], shp)
            return {"ewadd": s.add, "ewmul": s.mul, "ewdiv": s.div}[t](a, b)
        if t == "ewexp":
            return s.exp(ins[0])
        if t == "sqr":
            return s.mul(ins[0], ins[0])
        if t == "sqrt":
            return s.sqrt(ins[0])
        if t == "silu":
            return s.silu(ins[0])
        if t == "repeat":
            return s.broadcast(ins[0], tuple(out_shape))
        if t == "reshape":
            return s.reshape(ins[0], tuple(out_shape))
        raise ValueError(f"Unsupported: eval of {t}")

    def _graphdef(self, g, op, vals):
        """eval_core.hpp:226-241 — grid-major block order."""
        bg = op["blockGraph"]
        outs = [self.s.zeros(tuple(g["tensors"][t]["shape"])) for t in op["outputs"]]
        gx, gy, gz = bg["grid"]
        for bx in range(gx):
            for by in range(gy):
                for bz in range(gz):
                    self._block(g, op, bg, (bx, by, bz), vals, outs)
        for t, o in zip(op["outputs"], outs):
            vals[t] = o

    def _load_tile(self, dev, attrs, bc, bg, it):
        """eval_core.hpp:244-270"""
        s = self.s
        dshape = list(s.shape(dev))
        tile, off = list(dshape), [0] * len(dshape)
        imap = _dm(attrs["imap"], True)
        for a, t in enumerate(imap):
            if t == PHI:
                continue
            tile[t] //= bg["grid"][a]
            off[t] += bc[a] * tile[t]
        ft = _dm(attrs["fmap"], False)[0]
        if ft != PHI:
            tile[ft] //= bg["forloop"]
            off[ft] += it * tile[ft]
        sl = tuple(slice(o, o + d) for o, d in zip(off, tile))
        return s.copy(s.getitem(dev, sl))

    def _block(self, g, op, bg, bc, vals, outs):
        """eval_core.hpp:272-376"""
        s = self.s
        ops, T = bg["ops"], bg["tensors"]
        bvals = [None] * len(T)
        post = [False] * len(T)
        for bop in ops:  # :277-294
            if bop["type"] == "accum":
                post[bop["outputs"][0]] = True
                continue
            if bop["type"] in ("initer", "outsaver"):
                continue
            if any(post[t] for t in bop["inputs"]):
                post[bop["outputs"][0]] = True

        def is_post(bop):
            return any(post[t] for t in bop["inputs"])

        acc = {}
        for bop in ops:  # :296-301
            if bop["type"] == "accum":
                acc[bop["id"]] = s.zeros(tuple(T[bop["outputs"][0]]["shape"]))
        for it in range(bg["forloop"]):  # :303-341
            for bop in ops:
                typ = bop["type"]
                if typ == "initer":
                    a = bop["attrs"]
                    dev = vals[op["inputs"][a["operand"]]]
                    bvals[bop["outputs"][0]] = self._load_tile(dev, a, bc, bg, it)
                    continue
                if typ == "accum":
                    val = bvals[bop["inputs"][0]]
                    t = _dm(bop["attrs"]["fmap"], False)[0]
                    if t == PHI:
                        acc[bop["id"]] = s.add(acc[bop["id"]], val)
                    else:
                        d = s.shape(val)[t]
                        sl = tuple(slice(it * d, (it + 1) * d) if k == t else slice(None)
                                   for k in range(len(s.shape(val))))
                        s.setitem(acc[bop["id"]], sl, val)
                    continue
                if typ == "outsaver" or is_post(bop):
                    continue
                ins = [bvals[t] for t in bop["inputs"]]
                bvals[bop["outputs"][0]] = self._predef(bop, ins, T[bop["outputs"][0]]["shape"])
        for bop in ops:  # :344-346
            if bop["type"] == "accum":
                bvals[bop["outputs"][0]] = acc[bop["id"]]
        saver = 0
        for bop in ops:  # :348-375
            typ = bop["type"]
            if typ == "outsaver":
                val = bvals[bop["inputs"][0]]
                omap = _dm(bop["attrs"]["omap"], True)
                vs = s.shape(val)
                off = [0] * len(vs)
                for ax, t in enumerate(omap):
                    off[t] += bc[ax] * vs[t]
                sl = tuple(slice(o, o + d) for o, d in zip(off, vs))
                s.setitem(outs[saver], sl, val)
                saver += 1
                continue
            if typ in ("initer", "accum") or not is_post(bop):
                continue
            ins = [bvals[t] for t in bop["inputs"]]
            bvals[bop["outputs"][0]] = self._predef(bop, ins, T[bop["outputs"][0]]["shape"])


# ---------------------------------------------------------------------------
# Verifier (ffeval.cpp, equiv.cpp, stability.cpp)
# ---------------------------------------------------------------------------

def graph_has_silu(g) -> bool:
    """equiv.cpp:22-30"""
    for op in g["ops"]:
        if op["type"] == "silu":
            return True
        for bop in op.get("blockGraph", {}).get("ops", []):
            if bop["type"] == "silu":
                return True
    return False


def sample_inputs(field: Field, shapes, rng: Rng):
    """ffeval.cpp:29-40: per element xp = uniform(p) then xq = uniform(q)."""
    out = []
    for shp in shapes:
        n = int(np.prod(shp))
        xp, xq = rng.uniform_pairs(n, field.p, field.q)
        out.append((xp.reshape(shp), xq.reshape(shp), np.ones(shp, bool)))
    return out


def silu_tables(field: Field, rng: Rng):
    """ffeval.cpp:20-27: p draws uniform(p), then q draws uniform(q)."""
    return rng.uniform_many(field.p, field.p), rng.uniform_many(field.q, field.q)


def ff_attempt(g, seed, stream, field: Optional[Field] = None, with_silu=None):
    """One attempt for one graph as equiv.cpp:57-68 performs it."""
    field = field or Field()
    rng = Rng.derive(seed, stream)
    inputs = sample_inputs(field, [g["tensors"][t]["shape"] for t in g["inputs"]], rng)
    omega = field.sample_omega(rng)
    tabs = silu_tables(field, rng) if (graph_has_silu(g) if with_silu is None else with_silu) else None
    return inputs, omega, Evaluator(FFSem(field, omega, tabs)).run(g, inputs)


def random_test_equivalence(g1, g2, num_tests=1, seed=0, max_resamples=16,
                            field: Optional[Field] = None) -> dict:
    """equiv.cpp:34-94.  Returns the EquivVerdict fields as a dict
    (kind 0 Equivalent / 1 NotEquivalent / 2 Inconclusive)."""
    field = field or Field()
    if len(g1["inputs"]) != len(g2["inputs"]) or len(g1["outputs"]) != len(g2["outputs"]):
        raise ValueError("ShapeMismatch: graph arity")
    shapes = []
    for a, b in zip(g1["inputs"], g2["inputs"]):
        if g1["tensors"][a]["shape"] != g2["tensors"][b]["shape"]:
            raise ValueError("ShapeMismatch: input shapes")
        shapes.append(g1["tensors"][a]["shape"])
    for a, b in zip(g1["outputs"], g2["outputs"]):
        if g1["tensors"][a]["shape"] != g2["tensors"][b]["shape"]:
            raise ValueError("ShapeMismatch: output shapes")
    needs_silu = graph_has_silu(g1) or graph_has_silu(g2)
    v = dict(kind=0, rounds_run=0, resamples=0, has_witness=0, w_seed=0, w_round=0, w_omega=0,
             w_tensor=0, w_index=0)
    for rnd in range(num_tests):
        done = False
        for attempt in range(max_resamples + 1):
            rng = Rng.derive(seed, rnd * 131071 + attempt)
            inputs = sample_inputs(field, shapes, rng)
            omega = field.sample_omega(rng)
            tabs = silu_tables(field, rng) if needs_silu else None
            sem = FFSem(field, omega, tabs)
            try:
                o1 = Evaluator(sem).run(g1, inputs)
                o2 = Evaluator(sem).run(g2, inputs)
            except ResampleNeeded:
                v["resamples"] += 1
                continue
            for t, (a, b) in enumerate(zip(o1, o2)):
                ap, aq, ad = (x.reshape(-1) for x in a)
                bp, bq, bd = (x.reshape(-1) for x in b)
                bad = (ap != bp) | (ad & bd & (aq != bq))  # FFValue::operator== (field.hpp:41-45)
                if np.any(bad):
                    v.update(kind=1, has_witness=1, w_seed=seed, w_round=rnd, w_omega=omega,
                             w_tensor=t, w_index=int(np.argmax(bad)), rounds_run=rnd + 1)
                    return v
            done = True
            break
        if not done:
            v.update(kind=2, rounds_run=rnd)
            return v
    v.update(kind=0, rounds_run=num_tests)
    return v


def eval_mugraph(g, inputs: Sequence[np.ndarray]) -> List[np.ndarray]:
    """interp.cpp:29-34 (double precision)."""
    return Evaluator(FloatSem()).run(g, [np.asarray(x, np.float64) for x in inputs])


def float_stability_filter(g, program, trials=1, tol=1e-3, seed=17, scale=1.0) -> bool:
    """stability.cpp:25-50"""
    for trial in range(trials):
        rng = Rng.derive(seed, trial)
        ins = []
        for t in program["inputs"]:
            shp = program["tensors"][t]["shape"]
            ins.append(np.array([rng.normal() * scale for _ in range(int(np.prod(shp)))]).reshape(shp))
        ref = eval_mugraph(program, ins)
        out = eval_mugraph(g, ins)
        for r, o in zip(ref, out):
            if not np.all(np.isfinite(o)):
                return False
            if np.any(np.abs(o - r) / np.maximum(np.abs(r), 1e-6) > tol):
                return False
    return True

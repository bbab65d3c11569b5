"""µGraph construction API (Python mirror of the reference builder API).

Mirrors ``tpo::ir::GraphBuilder`` / ``tpo::ir::BlockBuilder``
(reference ``proj/core/include/tpo/ir/graph.hpp:105-136``,
``proj/core/src/graph.cpp:36-124``) and the JSON wire format of
``proj/core/src/serialize.cpp:40-266`` so that graphs authored here are read
unchanged by the reference (``kernel_graph_from_json``) and by this
package's C-ABI (``tpo_gpu_compile``).  Shape inference follows
``proj/core/src/shape_infer.cpp:27-179``; errors raise :class:`TpoError`
with the reference's ``ErrCode`` names.

A graph is a plain dict in wire format; builders only append to it.
"""
from __future__ import annotations

import enum
import json
from typing import Dict, List, Optional, Sequence

PHI = -1  # replica marker (reference kReplica, shape.hpp:89)


class ErrCode(enum.IntEnum):
    """Ordinals of ``tpo::ErrCode`` (reference shape.hpp:27-42)."""
    ShapeMismatch = 0
    NotDivisible = 1
    ReplicaInOmap = 2
    Unsupported = 3
    DivByZero = 4
    NonResidue = 5
    PoisonedExponent = 6
    BudgetExhausted = 7
    Infeasible = 8
    DoesNotFit = 9
    ParseError = 10
    NotLax = 11
    UnknownSuite = 12
    ConfigError = 13


class TpoError(RuntimeError):
    def __init__(self, code: ErrCode, msg: str = ""):
        super().__init__(f"{ErrCode(code).name}: {msg}")
        self.code = ErrCode(code)


class OpType(enum.IntEnum):
    """Operator set (reference ops.hpp:26-43), same ordinals and names."""
    InIter = 0
    OutSaver = 1
    Matmul = 2
    Sum = 3
    EwAdd = 4
    EwMul = 5
    EwDiv = 6
    EwExp = 7
    Repeat = 8
    Reshape = 9
    Sqr = 10
    Sqrt = 11
    SiLU = 12
    Accum = 13
    ConcatMatmul = 14
    GraphDef = 15


OP_NAMES = ["initer", "outsaver", "matmul", "sum", "ewadd", "ewmul", "ewdiv", "ewexp",
            "repeat", "reshape", "sqr", "sqrt", "silu", "accum", "concatmatmul", "graphdef"]
ELEMENTWISE = {OpType.EwAdd, OpType.EwMul, OpType.EwDiv, OpType.EwExp, OpType.Sqr,
               OpType.Sqrt, OpType.SiLU}  # ops.cpp:92-105
_GRID_AXES = ("x", "y", "z")


def op_from_name(name: str) -> OpType:
    try:
        return OpType(OP_NAMES.index(name))
    except ValueError:
        raise TpoError(ErrCode.ParseError, f"unknown op type '{name}'")


def _allowed_at(t: OpType, level: str) -> bool:
    # reference ops.cpp:38-60
    if t in (OpType.InIter, OpType.OutSaver, OpType.Accum):
        return level == "block"
    if t in (OpType.Matmul, OpType.Sum, OpType.EwAdd, OpType.EwMul, OpType.EwDiv, OpType.EwExp):
        return True
    if t == OpType.GraphDef:
        return level == "kernel"
    return level != "thread"


# ---- wire-format helpers -------------------------------------------------

def dimmap_to_json(m: Sequence[int], grid_axes: bool) -> dict:
    keys = _GRID_AXES if grid_axes else ("i",)
    return {keys[a]: ("phi" if t == PHI else int(t)) for a, t in enumerate(m)}


def dimmap_from_json(j: dict, grid_axes: bool) -> List[int]:
    out = []
    for k in (_GRID_AXES if grid_axes else ("i",)):
        if k not in j:
            break
        v = j[k]
        if isinstance(v, str):
            if v != "phi":
                raise TpoError(ErrCode.ParseError, "dim map entry must be an index or 'phi'")
            out.append(PHI)
        else:
            out.append(int(v))
    return out


# ---- shape inference (reference shape_infer.cpp) --------------------------

def broadcast_shapes(a: Sequence[int], b: Sequence[int]) -> Optional[List[int]]:
    r = max(len(a), len(b))
    out = []
    for i in range(r):
        da = 1 if i < r - len(a) else a[i - (r - len(a))]
        db = 1 if i < r - len(b) else b[i - (r - len(b))]
        if da != db and da != 1 and db != 1:
            return None
        out.append(max(da, db))
    return out


def _valid(s: Sequence[int]) -> bool:
    return 1 <= len(s) <= 4 and all(d >= 1 for d in s)


def _matmul_shape(a, b):
    if len(a) < 2 or len(b) < 2 or len(a) != len(b):
        raise TpoError(ErrCode.ShapeMismatch, "matmul rank")
    if list(a[:-2]) != list(b[:-2]) or a[-1] != b[-2]:
        raise TpoError(ErrCode.ShapeMismatch, "matmul dims")
    return list(a[:-1]) + [b[-1]]


def infer_output_shape(t: OpType, attrs: dict, ins: List[List[int]], level: str) -> List[int]:
    if not _allowed_at(t, level):
        raise TpoError(ErrCode.Unsupported, f"{OP_NAMES[t]} at {level} level")
    for s in ins:
        if not _valid(s):
            raise TpoError(ErrCode.ShapeMismatch, "invalid input shape")
    if t == OpType.Matmul:
        if len(ins) != 2:
            raise TpoError(ErrCode.ShapeMismatch, "arity")
        return _matmul_shape(ins[0], ins[1])
    if t == OpType.ConcatMatmul:
        if len(ins) != 4:
            raise TpoError(ErrCode.ShapeMismatch, "arity")
        wy, xz = _matmul_shape(ins[0], ins[2]), _matmul_shape(ins[1], ins[3])
        if wy != xz:
            raise TpoError(ErrCode.ShapeMismatch, "concatmatmul halves")
        return wy
    if t == OpType.Sum:
        d, g = attrs["dim"], attrs["group"]
        if len(ins) != 1 or not (0 <= d < len(ins[0])) or g < 1 or ins[0][d] % g:
            raise TpoError(ErrCode.ShapeMismatch, "sum")
        out = list(ins[0])
        out[d] //= g
        return out
    if t in (OpType.EwAdd, OpType.EwMul, OpType.EwDiv):
        if len(ins) != 2:
            raise TpoError(ErrCode.ShapeMismatch, "arity")
        s = broadcast_shapes(ins[0], ins[1])
        if s is None:
            raise TpoError(ErrCode.ShapeMismatch, "broadcast")
        return s
    if t in (OpType.EwExp, OpType.Sqr, OpType.Sqrt, OpType.SiLU):
        if len(ins) != 1:
            raise TpoError(ErrCode.ShapeMismatch, "arity")
        return list(ins[0])
    if t == OpType.Repeat:
        tgt = list(attrs["target"])
        s = broadcast_shapes(ins[0], tgt) if _valid(tgt) else None
        if s != tgt:
            raise TpoError(ErrCode.ShapeMismatch, "repeat")
        return tgt
    if t == OpType.Reshape:
        tgt = list(attrs["target"])
        if not _valid(tgt) or _prod(tgt) != _prod(ins[0]):
            raise TpoError(ErrCode.ShapeMismatch, "reshape")
        return tgt
    if t == OpType.Accum:
        fm = attrs["fmap"]
        if len(ins) != 1 or len(fm) != 1:
            raise TpoError(ErrCode.ShapeMismatch, "accum")
        if fm[0] != PHI and not (0 <= fm[0] < len(ins[0])):
            raise TpoError(ErrCode.ShapeMismatch, "accum dim")
        return list(ins[0])
    raise TpoError(ErrCode.Unsupported, OP_NAMES[t])


def _prod(s):
    n = 1
    for d in s:
        n *= d
    return n


def partition_shape(shape, dmap, extents):
    """reference shape_infer.cpp:151-166"""
    if len(dmap) != len(extents):
        raise TpoError(ErrCode.ShapeMismatch, "partition axes")
    used = [t for t in dmap if t != PHI]
    if len(set(used)) != len(used):
        raise TpoError(ErrCode.ShapeMismatch, "partition targets")
    out = list(shape)
    for t, e in zip(dmap, extents):
        if t == PHI:
            continue
        if not (0 <= t < len(shape)):
            raise TpoError(ErrCode.ShapeMismatch, "partition dim")
        if e < 1 or out[t] % e:
            raise TpoError(ErrCode.NotDivisible, f"partition {shape} by {dmap}/{extents}")
        out[t] //= e
    return out


def assemble_output_shape(per_block, omap, grid):
    """reference shape_infer.cpp:168-179"""
    if len(omap) != len(grid):
        raise TpoError(ErrCode.ShapeMismatch, "omap axes")
    used = [t for t in omap if t != PHI]
    if len(set(used)) != len(used):
        raise TpoError(ErrCode.ShapeMismatch, "omap targets")
    out = list(per_block)
    for t, g in zip(omap, grid):
        if t == PHI:
            raise TpoError(ErrCode.ReplicaInOmap, "replica in omap")
        if not (0 <= t < len(per_block)):
            raise TpoError(ErrCode.ShapeMismatch, "omap dim")
        out[t] *= g
    return out


# ---- builders --------------------------------------------------------------

def _attrs_json(t: OpType, attrs: Optional[dict]) -> dict:
    attrs = attrs or {}
    if t == OpType.Sum:
        return {"dim": int(attrs["dim"]), "group": int(attrs["group"])}
    if t == OpType.Accum:
        return {"fmap": dimmap_to_json(attrs.get("fmap", [PHI]), False)}
    if t in (OpType.Reshape, OpType.Repeat):
        return {"target": [int(d) for d in attrs["target"]]}
    return {}


class BlockBuilder:
    """reference graph.hpp:124-141, graph.cpp:76-124"""

    def __init__(self, grid: Sequence[int], forloop: int, operand_shapes: Sequence[Sequence[int]]):
        self.grid = [int(g) for g in grid]
        assert len(self.grid) == 3
        self.forloop = int(forloop)
        self.operand_shapes = [list(s) for s in operand_shapes]
        self.tensors: List[dict] = []
        self.ops: List[dict] = []
        self.out_shapes: List[List[int]] = []
        self.thread_groups: List[dict] = []

    def _shape(self, t):
        return self.tensors[t]["shape"]

    def _new_tensor(self, shape):
        tid = len(self.tensors)
        self.tensors.append({"id": tid, "shape": [int(d) for d in shape], "scope": "shared"})
        return tid

    def initer(self, operand: int, imap: Sequence[int], fmap: Sequence[int]) -> int:
        dev = self.operand_shapes[operand]
        ext = (self.grid + [1] * 3)[: len(imap)]
        tile = partition_shape(dev, list(imap), ext)
        tile = partition_shape(tile, list(fmap), [self.forloop])
        out = self._new_tensor(tile)
        self.ops.append({"id": len(self.ops), "type": "initer",
                         "attrs": {"operand": int(operand), "imap": dimmap_to_json(imap, True),
                                   "fmap": dimmap_to_json(fmap, False)},
                         "inputs": [], "outputs": [out]})
        return out

    def op(self, t: OpType, inputs: Sequence[int], attrs: Optional[dict] = None) -> int:
        t = OpType(t)
        shape = infer_output_shape(t, attrs or {}, [self._shape(i) for i in inputs], "block")
        if t == OpType.Accum:
            fm = (attrs or {}).get("fmap", [PHI])
            attrs = {"fmap": fm}
            if fm[0] != PHI:
                shape[fm[0]] *= self.forloop
        out = self._new_tensor(shape)
        self.ops.append({"id": len(self.ops), "type": OP_NAMES[t], "attrs": _attrs_json(t, attrs),
                         "inputs": [int(i) for i in inputs], "outputs": [out]})
        return out

    def outsaver(self, value: int, omap: Sequence[int]) -> List[int]:
        ext = (self.grid + [1] * 3)[: len(omap)]
        out = assemble_output_shape(self._shape(value), list(omap), ext)
        self.ops.append({"id": len(self.ops), "type": "outsaver",
                         "attrs": {"omap": dimmap_to_json(omap, True)},
                         "inputs": [int(value)], "outputs": []})
        self.out_shapes.append(out)
        return out

    def finish(self) -> dict:
        j = {"grid": list(self.grid), "forloop": self.forloop, "tensors": self.tensors,
             "ops": self.ops}
        if self.thread_groups:
            j["threadGroups"] = self.thread_groups
        return j


class GraphBuilder:
    """reference graph.hpp:105-121, graph.cpp:36-74"""

    def __init__(self):
        self.g = {"tensors": [], "ops": [], "inputs": [], "outputs": []}

    def _new_tensor(self, shape):
        tid = len(self.g["tensors"])
        self.g["tensors"].append({"id": tid, "shape": [int(d) for d in shape], "scope": "device"})
        return tid

    def shape(self, t: int) -> List[int]:
        return list(self.g["tensors"][t]["shape"])

    def input(self, shape: Sequence[int]) -> int:
        t = self._new_tensor(shape)
        self.g["inputs"].append(t)
        return t

    def op(self, t: OpType, inputs: Sequence[int], attrs: Optional[dict] = None) -> int:
        t = OpType(t)
        shape = infer_output_shape(t, attrs or {}, [self.shape(i) for i in inputs], "kernel")
        out = self._new_tensor(shape)
        self.g["ops"].append({"id": len(self.g["ops"]), "type": OP_NAMES[t],
                              "attrs": _attrs_json(t, attrs),
                              "inputs": [int(i) for i in inputs], "outputs": [out]})
        return out

    def graphdef(self, inputs: Sequence[int], block: BlockBuilder | dict,
                 out_shapes: Optional[Sequence[Sequence[int]]] = None) -> int:
        if isinstance(block, BlockBuilder):
            if out_shapes is None:
                out_shapes = block.out_shapes
            block = block.finish()
        outs = [self._new_tensor(s) for s in out_shapes]
        self.g["ops"].append({"id": len(self.g["ops"]), "type": "graphdef", "attrs": {},
                              "inputs": [int(i) for i in inputs], "outputs": outs,
                              "blockGraph": block})
        return outs[0]

    def finish(self, outputs: Sequence[int]) -> dict:
        self.g["outputs"] = [int(o) for o in outputs]
        return self.g


def to_json(g: dict) -> str:
    return json.dumps(g, separators=(",", ":"))


def input_shapes(g: dict) -> List[List[int]]:
    return [list(g["tensors"][t]["shape"]) for t in g["inputs"]]


def output_shapes(g: dict) -> List[List[int]]:
    return [list(g["tensors"][t]["shape"]) for t in g["outputs"]]


def has_silu(g: dict) -> bool:
    """reference equiv.cpp:22-30"""
    for op in g["ops"]:
        if op["type"] == "silu":
            return True
        for bop in op.get("blockGraph", {}).get("ops", []):
            if bop["type"] == "silu":
                return True
    return False

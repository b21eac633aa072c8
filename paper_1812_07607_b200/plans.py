"""Plan-file JSON surface: the reference's Python entry
points ``run_etl``, ``run_query``, ``collection_patches``,
``collection_stats`` and ``store_stats`` (bindings/py_module.cpp:139-335)
over the B200 operators.

* Plan files parse with the reference's strict schema
  (src/planfile.cpp:14-441): unknown keys, wrong types and unknown ops are
  ValidationError("plan file: ...") with the reference's messages.
* The ETL section (generator tiles | whole_image, transformers depth_proxy /
  color_histogram) reads the VideoStore through libpdb_cuda's reader and runs
  K1 over the decoded frames (pdb_store_featurize); patch ids, lineage,
  params digests and metadata are the reference's (src/core.cpp:78-138,
  src/etl.cpp:252-373), so the materialized collection file is
  byte-identical to PatchCollection::materialize's (src/etl.cpp:414-438,
  src/record_store.cpp, src/core.cpp:221-265).
* The plan runs on a materializing executor with the reference Volcano
  engine's emission order and id assignment (src/query.cpp:584-1029):
  scan, select, nl_join, sim_join (K2 + K3), dedup (csrc/dedup.cu), count_by.
  ``within`` predicates are evaluated on the GPU: cross-side atoms through
  the similarity join, same-side atoms through pdb_rows_within.
  index_join, backtrace and index builds / loads are outside the hot path
  (metadata / bbox indexes and frame re-reads) and raise
  UnsupportedError.
"""

from __future__ import annotations

import ctypes as C
import json
import os
import struct
import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _capi as capi
from . import patchdb as pdb
from .patchdb import (BoundingBox, ConfigError, DimensionMismatchError, Error, IoError,
                      LineageStep, Patch, ShapeError, TagMismatchError, ValidationError)


class UnsupportedError(ConfigError):
    """A plan feature outside the B200 build's scope."""


# ---------------------------------------------------------------------------
# Plan-file schema (src/planfile.cpp)


def _bad(msg: str):
    raise ValidationError("plan file: " + msg)


def _expect_object(j, where):
    if not isinstance(j, dict):
        _bad(where + " must be an object")


def _expect_keys(j, where, keys):
    _expect_object(j, where)
    for k in j:
        if k not in keys:
            _bad(f"{where}: unknown key '{k}'")


def _is_int(v) -> bool:
    return isinstance(v, int) and not isinstance(v, bool)


def _is_num(v) -> bool:
    return isinstance(v, (int, float)) and not isinstance(v, bool)


def _get_u64(v, where) -> int:
    if not _is_int(v) or v < 0:
        _bad(where + " must be a non-negative integer")
    return v


def _get_num(v, where) -> float:
    if not _is_num(v):
        _bad(where + " must be a number")
    return float(v)


def _get_str(v, where) -> str:
    if not isinstance(v, str):
        _bad(where + " must be a string")
    return v


def _meta_from_json(v, where):
    """planfile.cpp:54-77: numbers and strings map directly; four numbers
    are a box (a tuple here), an array of strings a string list."""
    if _is_int(v):
        return v
    if isinstance(v, float):
        return v
    if isinstance(v, str):
        return v
    if isinstance(v, list):
        if v and len(v) == 4 and all(_is_num(e) for e in v):
            return tuple(_get_u64(e, where) for e in v)
        return [_get_str(e, where + " element") for e in v]
    _bad(where + ": literal must be a number, string, box, or string list")


@dataclass
class Operand:
    literal: object = None
    slot: int = -1          # -1: literal
    key: str = ""

    def describe(self) -> str:
        return _meta_to_string(self.literal) if self.slot < 0 else f"s{self.slot}.{self.key}"


def _operand_from_json(j, where) -> Operand:
    _expect_object(j, where)
    if "lit" in j:
        _expect_keys(j, where, ("lit",))
        return Operand(literal=_meta_from_json(j["lit"], where + ".lit"))
    _expect_keys(j, where, ("slot", "key"))
    if "slot" not in j or "key" not in j:
        _bad(where + " needs either {lit} or {slot, key}")
    return Operand(slot=_get_u64(j["slot"], where + ".slot"), key=_get_str(j["key"], where + ".key"))


_CMP_NAMES = {"eq": "==", "ne": "!=", "lt": "<", "le": "<=", "gt": ">", "ge": ">="}


@dataclass
class Predicate:
    kind: str                       # cmp | within | contains | and | or | not
    op: str = ""                    # cmp: eq ne lt le gt ge
    lhs: Optional[Operand] = None
    rhs: Optional[Operand] = None
    offset: float = 0.0
    slot_a: int = 0
    slot_b: int = 0
    radius: float = 0.0
    key: str = ""                   # contains: list key
    needle: str = ""
    parts: List["Predicate"] = field(default_factory=list)

    def describe(self) -> str:
        """Predicate::describe (src/query.cpp:239-267)."""
        k = self.kind
        if k == "cmp":
            s = f"{self.lhs.describe()} {_CMP_NAMES[self.op]} {self.rhs.describe()}"
            if self.offset != 0.0:
                s += " + " + _fmt(self.offset)
            return s
        if k == "within":
            return f"dist(s{self.slot_a};s{self.slot_b}) <= {_fmt(self.radius)}"
        if k == "contains":
            return f"contains(s{self.slot_a}.{self.key}; '{self.needle}')"
        if k in ("and", "or"):
            j = " AND " if k == "and" else " OR "
            return "(" + j.join(c.describe() for c in self.parts) + ")"
        return "NOT " + (self.parts[0].describe() if self.parts else "()")


def _pred_from_json(j, where) -> Predicate:
    """planfile.cpp:100-150."""
    _expect_object(j, where)
    if "kind" not in j:
        _bad(where + " needs a kind")
    kind = _get_str(j["kind"], where + ".kind")
    if kind == "cmp":
        _expect_keys(j, where, ("kind", "op", "lhs", "rhs", "offset"))
        if "op" not in j or "lhs" not in j or "rhs" not in j:
            _bad(where + ": cmp needs op, lhs, rhs")
        offset = _get_num(j["offset"], where + ".offset") if "offset" in j else 0.0
        name = _get_str(j["op"], where + ".op")
        if name not in _CMP_NAMES:
            _bad(f"{where}: unknown comparison '{name}'")
        return Predicate("cmp", op=name, lhs=_operand_from_json(j["lhs"], where + ".lhs"),
                         rhs=_operand_from_json(j["rhs"], where + ".rhs"), offset=offset)
    if kind == "within":
        _expect_keys(j, where, ("kind", "slot_a", "slot_b", "radius"))
        if "slot_a" not in j or "slot_b" not in j or "radius" not in j:
            _bad(where + ": within needs slot_a, slot_b, radius")
        return Predicate("within", slot_a=_get_u64(j["slot_a"], where + ".slot_a"),
                         slot_b=_get_u64(j["slot_b"], where + ".slot_b"),
                         radius=_get_num(j["radius"], where + ".radius"))
    if kind == "contains":
        _expect_keys(j, where, ("kind", "slot", "key", "value"))
        if "slot" not in j or "key" not in j or "value" not in j:
            _bad(where + ": contains needs slot, key, value")
        return Predicate("contains", slot_a=_get_u64(j["slot"], where + ".slot"),
                         key=_get_str(j["key"], where + ".key"),
                         needle=_get_str(j["value"], where + ".value"))
    if kind in ("and", "or"):
        _expect_keys(j, where, ("kind", "parts"))
        if "parts" not in j or not isinstance(j["parts"], list):
            _bad(f"{where}: {kind} needs a parts array")
        return Predicate(kind, parts=[_pred_from_json(p, f"{where}.parts[{i}]")
                                      for i, p in enumerate(j["parts"])])
    if kind == "not":
        _expect_keys(j, where, ("kind", "part"))
        if "part" not in j:
            _bad(where + ": not needs a part")
        return Predicate("not", parts=[_pred_from_json(j["part"], where + ".part")])
    _bad(f"{where}: unknown predicate kind '{kind}'")


@dataclass
class PlanNode:
    kind: str
    children: List["PlanNode"] = field(default_factory=list)
    collection: str = ""
    pred: Optional[Predicate] = None
    tau: float = 0.1
    side: pdb.BuildSide = pdb.BuildSide.automatic
    key: str = ""
    op_index: int = -1

    def label(self) -> str:
        """Compiler::label_of (src/query.cpp:626-649)."""
        k = self.kind
        if k == "scan":
            return f"Scan({self.collection})"
        if k == "select":
            return f"Select({self.pred.describe()})"
        if k == "nl_join":
            return f"NLJoin({self.pred.describe()})"
        if k == "sim_join":
            side = {0: "auto", 1: "left", 2: "right"}[int(self.side)]
            return f"SimJoin(tau={_fmt(self.tau)};build={side})"
        if k == "dedup":
            return f"Dedup(tau={_fmt(self.tau)})"
        if k == "count_by":
            return f"CountBy({self.key})"
        return k


def _plan_from_json(j, where) -> PlanNode:
    """planfile.cpp:152-254."""
    _expect_object(j, where)
    if "op" not in j:
        _bad(where + " needs an op")
    op = _get_str(j["op"], where + ".op")

    def child(key):
        if key not in j:
            _bad(f"{where}: {op} needs a '{key}' input")
        return _plan_from_json(j[key], f"{where}.{key}")

    if op == "scan":
        _expect_keys(j, where, ("op", "collection"))
        if "collection" not in j:
            _bad(where + ": scan needs a collection")
        return PlanNode("scan", collection=_get_str(j["collection"], where + ".collection"))
    if op == "select":
        _expect_keys(j, where, ("op", "input", "pred"))
        if "pred" not in j:
            _bad(where + ": select needs a pred")
        c = child("input")
        return PlanNode("select", [c], pred=_pred_from_json(j["pred"], where + ".pred"))
    if op == "nl_join":
        _expect_keys(j, where, ("op", "left", "right", "on"))
        if "on" not in j:
            _bad(where + ": nl_join needs an 'on' predicate")
        l, r = child("left"), child("right")
        return PlanNode("nl_join", [l, r], pred=_pred_from_json(j["on"], where + ".on"))
    if op == "index_join":
        _expect_keys(j, where, ("op", "left", "collection", "index", "probe_slot", "probe_key",
                                "mode", "key_offset", "range_lo", "range_hi"))
        raise UnsupportedError(f"{where}: index_join (metadata indexes) is outside the B200 "
                               "build's scope")
    if op == "sim_join":
        _expect_keys(j, where, ("op", "left", "right", "tau", "build_side"))
        if "tau" not in j:
            _bad(where + ": sim_join needs tau")
        side = pdb.BuildSide.automatic
        if "build_side" in j:
            s = _get_str(j["build_side"], where + ".build_side")
            if s not in ("automatic", "left", "right"):
                _bad(f"{where}: unknown build side '{s}'")
            side = pdb.BuildSide[s]
        l, r = child("left"), child("right")
        return PlanNode("sim_join", [l, r], tau=_get_num(j["tau"], where + ".tau"), side=side)
    if op == "dedup":
        _expect_keys(j, where, ("op", "input", "tau"))
        if "tau" not in j:
            _bad(where + ": dedup needs tau")
        c = child("input")
        return PlanNode("dedup", [c], tau=_get_num(j["tau"], where + ".tau"))
    if op == "count_by":
        _expect_keys(j, where, ("op", "input", "key"))
        if "key" not in j:
            _bad(where + ": count_by needs a key")
        c = child("input")
        return PlanNode("count_by", [c], key=_get_str(j["key"], where + ".key"))
    if op == "backtrace":
        _expect_keys(j, where, ("op", "input", "mode", "trace_slot"))
        raise UnsupportedError(f"{where}: backtrace (frame re-reads) is outside the B200 "
                               "build's scope")
    _bad(f"{where}: unknown op '{op}'")


@dataclass
class GeneratorSpec:
    kind: str = "whole_image"
    tile_w: int = 0
    tile_h: int = 0
    palette: list = field(default_factory=list)
    min_area: int = 1
    label_noise_p: float = 0.0
    seed: int = 0

    def validate(self) -> None:
        """GeneratorSpec::validate (src/etl.cpp:45-62)."""
        if self.kind == "tiles":
            if self.tile_w < 1 or self.tile_h < 1:
                raise ConfigError("tiles generator needs tile_w and tile_h >= 1")
        elif self.kind == "blob_detector":
            if not self.palette:
                raise ConfigError("blob_detector palette must not be empty")
            if self.min_area < 1:
                raise ConfigError("blob_detector min_area must be >= 1")
            if self.label_noise_p < 0.0 or self.label_noise_p > 1.0:
                raise ConfigError("label_noise_p must be within [0, 1]")


_GENERATORS = ("whole_image", "tiles", "blob_detector", "glyph_reader")
_TRANSFORMERS = ("color_histogram", "depth_proxy")


@dataclass
class TransformerSpec:
    kind: str = "color_histogram"
    bins: int = 8

    def validate(self) -> None:
        if self.kind == "color_histogram" and self.bins < 2:
            raise ConfigError("color_histogram needs at least 2 bins per channel")


def _generator_from_json(j, where) -> GeneratorSpec:
    """planfile.cpp:278-298 (+ palette 256-276)."""
    _expect_keys(j, where, ("kind", "tile_w", "tile_h", "palette", "min_area", "label_noise_p",
                            "seed"))
    if "kind" not in j:
        _bad(where + " needs a kind")
    g = GeneratorSpec()
    g.kind = _get_str(j["kind"], where + ".kind")
    if g.kind not in _GENERATORS:
        raise ConfigError(f"unknown generator kind '{g.kind}'")
    if "tile_w" in j:
        g.tile_w = _get_u64(j["tile_w"], where + ".tile_w") & 0xFFFFFFFF
    if "tile_h" in j:
        g.tile_h = _get_u64(j["tile_h"], where + ".tile_h") & 0xFFFFFFFF
    if "palette" in j:
        pw = where + ".palette"
        if not isinstance(j["palette"], list):
            _bad(pw + " must be an array of [r,g,b,label] entries")
        for i, e in enumerate(j["palette"]):
            ew = f"{pw}[{i}]"
            if not isinstance(e, list) or len(e) != 4:
                _bad(ew + " must be [r,g,b,label]")
            rgb = [_get_u64(e[c], ew) for c in range(3)]
            if any(v > 255 for v in rgb):
                _bad(ew + ": channel above 255")
            g.palette.append((*rgb, _get_str(e[3], ew + " label")))
    if "min_area" in j:
        g.min_area = _get_u64(j["min_area"], where + ".min_area") & 0xFFFFFFFF
    if "label_noise_p" in j:
        g.label_noise_p = _get_num(j["label_noise_p"], where + ".label_noise_p")
    if "seed" in j:
        g.seed = _get_u64(j["seed"], where + ".seed")
    return g


def _transformer_from_json(j, where) -> TransformerSpec:
    """planfile.cpp:300-308."""
    _expect_keys(j, where, ("kind", "bins"))
    if "kind" not in j:
        _bad(where + " needs a kind")
    t = TransformerSpec()
    t.kind = _get_str(j["kind"], where + ".kind")
    if t.kind not in _TRANSFORMERS:
        raise ConfigError(f"unknown transformer kind '{t.kind}'")
    if "bins" in j:
        t.bins = _get_u64(j["bins"], where + ".bins") & 0xFFFFFFFF
    return t


@dataclass
class EtlSection:
    name: str = "etl"
    store: str = ""
    generator: GeneratorSpec = field(default_factory=GeneratorSpec)
    transformers: List[TransformerSpec] = field(default_factory=list)
    output: str = ""


@dataclass
class PlanFile:
    stores: Dict[str, str] = field(default_factory=dict)
    collections: Dict[str, str] = field(default_factory=dict)
    etl: Optional[EtlSection] = None
    index_builds: list = field(default_factory=list)
    load_indexes: list = field(default_factory=list)
    plan: Optional[PlanNode] = None
    output: dict = field(default_factory=dict)


def _alias_map(j, where) -> Dict[str, str]:
    _expect_object(j, where)
    return {k: _get_str(v, f"{where}.{k}") for k, v in sorted(j.items())}


def parse_plan(text: str) -> PlanFile:
    """PlanFile::parse (src/planfile.cpp:372-441)."""
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        _bad(str(e))
    _expect_keys(j, "plan file", ("stores", "collections", "etl", "indexes", "load_indexes",
                                  "plan", "output"))
    pf = PlanFile()
    if "stores" in j:
        pf.stores = _alias_map(j["stores"], "stores")
    if "collections" in j:
        pf.collections = _alias_map(j["collections"], "collections")
    if "etl" in j:
        e = j["etl"]
        _expect_keys(e, "etl", ("name", "store", "generator", "transformers", "output"))
        if "store" not in e or "generator" not in e or "output" not in e:
            _bad("etl needs store, generator, output")
        s = EtlSection()
        if "name" in e:
            s.name = _get_str(e["name"], "etl.name")
        s.store = _get_str(e["store"], "etl.store")
        s.generator = _generator_from_json(e["generator"], "etl.generator")
        if "transformers" in e:
            if not isinstance(e["transformers"], list):
                _bad("etl.transformers must be an array")
            s.transformers = [_transformer_from_json(t, f"etl.transformers[{i}]")
                              for i, t in enumerate(e["transformers"])]
        s.output = _get_str(e["output"], "etl.output")
        pf.etl = s
    if "indexes" in j:
        if not isinstance(j["indexes"], list):
            _bad("indexes must be an array")
        for i, e in enumerate(j["indexes"]):
            w = f"indexes[{i}]"
            _expect_keys(e, w, ("collection", "name", "kind", "key", "leaf_size", "capacity"))
            if "name" not in e or "kind" not in e:
                _bad(w + " needs name and kind")
            pf.index_builds.append(e)
    if "load_indexes" in j:
        if not isinstance(j["load_indexes"], list):
            _bad("load_indexes must be an array")
        for i, e in enumerate(j["load_indexes"]):
            w = f"load_indexes[{i}]"
            _expect_keys(e, w, ("collection", "name"))
            if "collection" not in e or "name" not in e:
                _bad(w + " needs collection and name")
            pf.load_indexes.append(e)
    if "plan" in j:
        pf.plan = _plan_from_json(j["plan"], "plan")
    if "output" in j:
        _expect_keys(j["output"], "output", ("results", "stats_csv"))
        pf.output = dict(j["output"])
    return pf


def _collect_labels(p: Predicate, out: list) -> None:
    """collect_pred_labels (src/planfile.cpp:336-362)."""
    if p.kind == "cmp":
        for a, b in ((p.lhs, p.rhs), (p.rhs, p.lhs)):
            if a.slot >= 0 and a.key == "label" and b.slot < 0 and isinstance(b.literal, str):
                out.append(b.literal)
    elif p.kind == "contains":
        if p.key == "group_labels":
            out.append(p.needle)
    elif p.kind in ("and", "or", "not"):
        for c in p.parts:
            _collect_labels(c, out)


def _collect_plan_labels(n: PlanNode, out: list) -> None:
    if n.kind in ("select", "nl_join"):
        _collect_labels(n.pred, out)
    for c in n.children:
        _collect_plan_labels(c, out)


def check_stages(pf: PlanFile) -> None:
    """plan_stages + validate_pipeline (src/planfile.cpp:452-466,
    src/etl.cpp:533-594), joined as py_module.cpp:54-66 does."""
    if pf.etl is None:
        return
    viol = []
    g = pf.etl.generator
    schema_shape = None      # None: wildcard
    domain = None
    try:
        g.validate()
        if g.kind == "tiles":
            schema_shape = (g.tile_h, g.tile_w, 3)
        elif g.kind == "glyph_reader":
            schema_shape = (4, 16, 3)
        elif g.kind == "blob_detector":
            domain = {e[3] for e in g.palette}
    except ConfigError as e:
        viol.append((0, str(e)))
    for i, t in enumerate(pf.etl.transformers, start=1):
        try:
            t.validate()
        except ConfigError as e:
            viol.append((i, str(e)))
            continue
        if schema_shape is not None and not (len(schema_shape) == 3 and schema_shape[2] == 3):
            viol.append((i, f"{t.kind} requires pixel shaped input [h,w,3]"))
        if t.kind == "color_histogram":
            schema_shape = (3 * t.bins,)
    labels: list = []
    if pf.plan is not None:
        _collect_plan_labels(pf.plan, labels)
    for k, l in enumerate(labels, start=1 + len(pf.etl.transformers)):
        if domain is not None and l not in domain:
            viol.append((k, f"label '{l}' is not producible by this pipeline"))
    if viol:
        raise ValidationError("; ".join(f"stage {i}: {m}" for i, m in viol))


# ---------------------------------------------------------------------------
# Canonical patch serialization (src/core.cpp:165-265) and the record store
# (src/record_store.cpp): big-endian, values appended, sorted index + footer.

_FILE_MAGIC = b"PDBS0001"
_FOOTER_MAGIC = b"PDBSIDX1"
_COLLECTION_KEY = b"\xffcollection"
_FORWARD_KEY = b"\xfflineage_fwd"


def _tag(v) -> int:
    if isinstance(v, (bool, np.bool_)):
        raise TagMismatchError("boolean metadata values are not representable")
    if isinstance(v, (int, np.integer)):
        return 0
    if isinstance(v, (float, np.floating)):
        return 1
    if isinstance(v, str):
        return 2
    if isinstance(v, (tuple, BoundingBox)):
        return 3
    return 4


_TAG_NAMES = ("int", "float", "str", "box", "str_list")


def _box(v) -> Tuple[int, int, int, int]:
    if isinstance(v, BoundingBox):
        return (v.x1, v.y1, v.x2, v.y2)
    return tuple(int(x) for x in v)


def _str8(s: str) -> bytes:
    b = s.encode()
    if len(b) > 255:
        raise Error("string too long for u8 length prefix")
    return bytes([len(b)]) + b


def _str16(s: str) -> bytes:
    b = s.encode()
    return struct.pack(">H", len(b)) + b


def _ser_meta(v) -> bytes:
    t = _tag(v)
    out = bytes([t])
    if t == 0:
        return out + struct.pack(">q", int(v))
    if t == 1:
        return out + struct.pack(">d", float(v))
    if t == 2:
        return out + _str16(v)
    if t == 3:
        return out + struct.pack(">4I", *_box(v))
    return out + struct.pack(">H", len(v)) + b"".join(_str16(s) for s in v)


def _meta_keys(meta: dict) -> List[str]:
    return sorted(meta, key=lambda k: k.encode())   # std::map<std::string> order


def serialize_patch(p: Patch) -> bytes:
    """serialize_patch (src/core.cpp:221-265): u32 length + body."""
    data = np.ascontiguousarray(np.asarray(p.data, dtype=np.float32).ravel())
    body = [struct.pack(">QB", p.patch_id, len(p.shape)),
            struct.pack(f">{len(p.shape)}I", *p.shape), data.astype(">f4").tobytes(),
            struct.pack(">H", len(p.lineage))]
    for st in p.lineage:
        body.append(_str8(st.op_name))
        if isinstance(st.source, tuple):
            body.append(b"\x00" + _str8(st.source[0]) + struct.pack(">Q", st.source[1]))
        else:
            body.append(b"\x01" + struct.pack(">Q", st.source))
        if st.region is not None:
            body.append(b"\x01" + struct.pack(">4I", *_box(st.region)))
        else:
            body.append(b"\x00")
        body.append(struct.pack(">Q", st.params_digest))
    body.append(struct.pack(">H", len(p.meta)))
    for k in _meta_keys(p.meta):
        body.append(_str8(k) + _ser_meta(p.meta[k]))
    b = b"".join(body)
    return struct.pack(">I", len(b)) + b


class _Reader:
    def __init__(self, buf: bytes, pos: int = 0):
        self.b, self.p = buf, pos

    def take(self, fmt: str):
        v = struct.unpack_from(fmt, self.b, self.p)
        self.p += struct.calcsize(fmt)
        return v

    def u8(self):
        return self.take(">B")[0]

    def u16(self):
        return self.take(">H")[0]

    def u32(self):
        return self.take(">I")[0]

    def u64(self):
        return self.take(">Q")[0]

    def str8(self):
        n = self.u8()
        s = self.b[self.p:self.p + n].decode()
        self.p += n
        return s

    def str16(self):
        n = self.u16()
        s = self.b[self.p:self.p + n].decode()
        self.p += n
        return s


def deserialize_patch(rec: bytes) -> Patch:
    """deserialize_patch (src/core.cpp:267-330)."""
    r = _Reader(rec)
    if r.u32() != len(rec) - 4:
        raise Error("patch record length prefix does not match payload")
    pid = r.u64()
    rank = r.u8()
    shape = r.take(f">{rank}I") if rank else ()
    n = int(np.prod(shape)) if rank else 1
    data = np.frombuffer(rec, dtype=">f4", count=n, offset=r.p).astype(np.float32)
    r.p += 4 * n
    lineage = []
    for _ in range(r.u16()):
        op = r.str8()
        if r.u8() == 0:
            vid = r.str8()
            src = (vid, r.u64())
        else:
            src = r.u64()
        region = BoundingBox(*r.take(">4I")) if r.u8() else None
        lineage.append(LineageStep(op, src, region, r.u64()))
    meta = {}
    for _ in range(r.u16()):
        k = r.str8()
        t = r.u8()
        if t == 0:
            meta[k] = r.take(">q")[0]
        elif t == 1:
            meta[k] = r.take(">d")[0]
        elif t == 2:
            meta[k] = r.str16()
        elif t == 3:
            meta[k] = r.take(">4I")
        elif t == 4:
            meta[k] = [r.str16() for _ in range(r.u16())]
        else:
            raise Error("unknown metadata tag byte")
    if r.p != len(rec):
        raise Error("trailing bytes after patch record")
    return Patch(pid, data.reshape(shape) if rank else data, tuple(shape), meta, lineage)


def _serialize_forward(fwd: Dict[Tuple[str, int], List[int]]) -> bytes:
    """serialize_forward (src/etl.cpp:384-395): frames in FrameId order."""
    out = [struct.pack(">Q", len(fwd))]
    for (vid, fno) in sorted(fwd, key=lambda f: (f[0].encode(), f[1])):
        ids = fwd[(vid, fno)]
        out.append(_str8(vid) + struct.pack(">QI", fno, len(ids)) +
                   np.asarray(ids, dtype=">u8").tobytes())
    return b"".join(out)


def _write_store(path: str, values: List[bytes], keys: List[bytes]) -> int:
    """RecordStore::create + put... + finalize: values in put order, the
    index sorted by key.  Returns the file size."""
    try:
        f = open(path, "wb")
    except OSError:
        raise IoError("cannot open record store at " + path)
    with f:
        f.write(_FILE_MAGIC)
        pos = len(_FILE_MAGIC)
        index = {}
        for k, v in zip(keys, values):
            f.write(v)
            index[k] = (pos, len(v))
            pos += len(v)
        ent = [struct.pack(">I", len(k)) + k + struct.pack(">QQ", *index[k])
               for k in sorted(index)]
        f.write(b"".join(ent) + struct.pack(">QQ", pos, len(index)) + _FOOTER_MAGIC)
        return f.tell()


def _read_store(path: str) -> Tuple[bytes, Dict[bytes, Tuple[int, int]]]:
    """RecordStore::open + load_index (src/record_store.cpp:54-100)."""
    try:
        with open(path, "rb") as f:
            buf = f.read()
    except OSError:
        raise IoError("cannot open record store at " + path)
    if len(buf) < 8 + 24:
        raise IoError(f"record store {path} is truncated")
    if buf[:8] != _FILE_MAGIC:
        raise IoError(f"record store {path} has a bad file magic")
    if buf[-8:] != _FOOTER_MAGIC:
        raise IoError(f"record store {path} has a bad footer magic")
    index_off, n = struct.unpack_from(">QQ", buf, len(buf) - 24)
    if index_off < 8 or index_off > len(buf) - 24:
        raise IoError(f"record store {path} has a corrupt index offset")
    r = _Reader(buf, index_off)
    index = {}
    for _ in range(n):
        kl = r.u32()
        k = buf[r.p:r.p + kl]
        r.p += kl
        index[k] = r.take(">QQ")
    return buf, index


# ---------------------------------------------------------------------------
# Patch collections (src/etl.cpp:378-500)


class PatchCollection:
    """A materialized collection: the record-store file on disk plus the
    patches held in memory for the executor (scan order = key order =
    ascending patch id, as RecordStore::scan returns them)."""

    def __init__(self, path: str, patches: List[Patch], fwd: dict, size: int,
                 index_names: Sequence[str] = (), record_bytes: int = 0):
        self._path = path
        self.record_bytes = record_bytes   # sum of patch record sizes (scan's bytes_read)
        self.patches = patches
        self.fwd = fwd
        self.size = size
        self.index_names = list(index_names)

    def path(self) -> str:
        return self._path

    def patch_count(self) -> int:
        return len(self.patches)

    @staticmethod
    def _finish(path, patches, records: List[bytes]) -> "PatchCollection":
        fwd: Dict[Tuple[str, int], List[int]] = {}
        seen = set()
        for p in patches:
            if p.patch_id in seen:
                raise pdb.DuplicatePatchIdError(f"patch id {p.patch_id} materialized twice")
            seen.add(p.patch_id)
            for st in _base_frames(p):
                fwd.setdefault(st, []).append(p.patch_id)
        for ids in fwd.values():
            ids.sort()
        desc = b"PCOL" + struct.pack(">Q", len(patches))
        keys = [struct.pack(">Q", p.patch_id) for p in patches] + [_COLLECTION_KEY, _FORWARD_KEY]
        size = _write_store(path, records + [desc, _serialize_forward(fwd)], keys)
        order = sorted(range(len(patches)), key=lambda k: patches[k].patch_id)
        return PatchCollection(path, [patches[k] for k in order], fwd, size,
                               record_bytes=sum(len(r) for r in records))

    @classmethod
    def materialize(cls, patches: Sequence[Patch], path: str) -> "PatchCollection":
        """PatchCollection::materialize (src/etl.cpp:414-438)."""
        patches = list(patches)
        return cls._finish(path, patches, [serialize_patch(p) for p in patches])

    @classmethod
    def open(cls, path: str) -> "PatchCollection":
        """PatchCollection::open + load_all (src/etl.cpp:440-463)."""
        buf, index = _read_store(path)
        desc = index.get(_COLLECTION_KEY)
        if desc is None or desc[1] < 12 or buf[desc[0]:desc[0] + 4] != b"PCOL":
            raise IoError(path + " is not a patch collection")
        fwd = {}
        if _FORWARD_KEY in index:
            off, ln = index[_FORWARD_KEY]
            r = _Reader(buf[off:off + ln])
            for _ in range(r.u64()):
                vid = r.str8()
                fno, k = r.take(">QI")
                fwd[(vid, fno)] = list(r.take(f">{k}Q")) if k else []
        keys = sorted(k for k in index if k < b"\xff")
        patches = [deserialize_patch(buf[index[k][0]:index[k][0] + index[k][1]]) for k in keys]
        names = sorted(k[5:].decode() for k in index if k.startswith(b"\xffidx:"))
        return cls(path, patches, fwd, len(buf), names,
                   record_bytes=sum(index[k][1] for k in keys))


def _base_frames(p: Patch) -> List[Tuple[str, int]]:
    """base_frames_of (src/core.cpp:140-148)."""
    if not p.lineage or not isinstance(p.lineage[-1].source, tuple):
        raise pdb.MalformedLineageError(
            f"patch {p.patch_id}: lineage does not terminate in a base frame")
    return [tuple(st.source) for st in p.lineage if isinstance(st.source, tuple)]


# ---------------------------------------------------------------------------
# ETL on the B200 (generate + transform + materialize, columnar)


class _Columns:
    """Fixed-layout records as one numpy structured array: constant byte
    runs and big-endian columns, concatenated without padding."""

    def __init__(self):
        self.fields: List[Tuple[str, object]] = []

    def const(self, b: bytes):
        if self.fields and isinstance(self.fields[-1][1], bytes) and self.fields[-1][0] == "c":
            self.fields[-1] = ("c", self.fields[-1][1] + b)
        else:
            self.fields.append(("c", b))

    def col(self, dtype, arr):
        self.fields.append((dtype, arr))

    def build(self, n: int) -> np.ndarray:
        spec = []
        for k, (dt, v) in enumerate(self.fields):
            if dt == "c":
                spec.append((f"f{k}", f"S{len(v)}"))
            elif isinstance(v, np.ndarray) and v.ndim == 2:
                spec.append((f"f{k}", dt, (v.shape[1],)))
            else:
                spec.append((f"f{k}", dt))
        rec = np.empty(n, dtype=np.dtype(spec))
        for k, (dt, v) in enumerate(self.fields):
            rec[f"f{k}"] = v
        return rec


def _digest(op: str, params=()) -> int:
    return pdb._fnv_digest(op, list(params))


def _etl_histograms(vs: "pdb.VideoStore", th: int, tw: int, bins: int) -> np.ndarray:
    """Decode + K1 over every frame: host features [F * T, 3 * bins]."""
    import torch
    if not torch.cuda.is_available():
        raise pdb.DeviceError("NoDevice: no CUDA device visible (K1 has no CPU path)")
    feats = vs.featurize(th, tw, bins, "per_channel")
    return feats.cpu().numpy()


def materialize_etl(pf: PlanFile) -> PatchCollection:
    """materialize_etl (bindings/py_module.cpp:68-77) on the B200: VideoStore
    frames -> tiles / whole_image patches -> transformers -> collection."""
    etl = pf.etl
    store_path = pf.stores.get(etl.store, etl.store)
    vs = pdb.VideoStore.open(store_path)
    try:
        return _materialize(vs, etl)
    finally:
        vs.close()


def _materialize(vs, etl: EtlSection) -> PatchCollection:
    g = etl.generator
    g.validate()
    for t in etl.transformers:
        t.validate()
    if g.kind not in ("tiles", "whole_image"):
        raise UnsupportedError(f"generator '{g.kind}' is outside the B200 build's scope "
                               "(tiles and whole_image feed K1)")
    F, H, W, vid = vs.frame_count, vs.height, vs.width, vs.video_id
    if g.kind == "tiles":
        th, tw = g.tile_h, g.tile_w
        ntx, nty = W // tw, H // th
    else:
        th, tw, ntx, nty = H, W, 1, 1
    T = ntx * nty
    n = F * T
    chain = etl.transformers
    m = len(chain)
    base = pdb._Ids.next_id
    # the collection file is created before the first patch is pulled
    try:
        open(etl.output, "wb").close()
    except OSError:
        raise IoError("cannot open record store at " + etl.output)
    # the streaming pipeline stops at the first transformer applied to a
    # non-pixel patch: patch 0's chain, ids base .. base + j - 1 consumed
    for j, t in enumerate(chain, start=1):
        if any(c.kind == "color_histogram" for c in chain[:j - 1]):
            if n == 0:
                break
            pdb._Ids.next_id = base + j
            raise ShapeError(f"transformer input must be pixel shaped [h,w,3], patch "
                             f"{base + j - 1} is not")
    hist = next((t for t in chain if t.kind == "color_histogram"), None)
    depth = any(t.kind == "depth_proxy" for t in chain)

    k = np.arange(n, dtype=np.int64)
    fno = (k // T).astype(np.uint64)
    tix = k % T
    x1 = ((tix % ntx) * tw).astype(np.uint32)
    y1 = ((tix // ntx) * th).astype(np.uint32)
    x2, y2 = x1 + np.uint32(tw), y1 + np.uint32(th)
    ids = (base + k * (m + 1)).astype(np.uint64)       # make_patch ids
    pdb._Ids.next_id = base + n * (m + 1)
    final_ids = ids + np.uint64(m)
    reg_digest = np.array([_digest("make_patch", [("x1", int(a)), ("y1", int(b)),
                                                  ("x2", int(c)), ("y2", int(d))])
                           for a, b, c, d in zip(x1[:T], y1[:T], x2[:T], y2[:T])],
                          dtype=np.uint64)
    reg_digest = np.tile(reg_digest, F)
    depth_v = 1.0 - y2.astype(np.float64) / float(H) if depth else None

    if hist is not None:
        data = _etl_histograms(vs, th, tw, hist.bins) if n else \
            np.zeros((0, 3 * hist.bins), np.float32)
        shape = (3 * hist.bins,)
    else:
        frames = vs.scan_array() if n else np.zeros((0, H, W, 3), np.uint8)
        crop = frames[:, :nty * th, :ntx * tw, :].reshape(F, nty, th, ntx, tw, 3)
        data = crop.transpose(0, 1, 3, 2, 4, 5).reshape(n, th, tw, 3).astype(np.float32)
        shape = (th, tw, 3)
    flat = data.reshape(n, int(np.prod(shape)))

    # records (serialize_patch layout)
    c = _Columns()
    c.col(">u4", 0)
    c.col(">u8", final_ids)
    c.const(struct.pack(">B", len(shape)) + struct.pack(f">{len(shape)}I", *shape))
    c.col(">f4", flat)
    c.const(struct.pack(">H", m + 1))
    for j in range(m, 0, -1):
        t = chain[j - 1]
        c.const(_str8(t.kind) + b"\x01")
        c.col(">u8", ids + np.uint64(j - 1))
        dg = _digest("color_histogram", [("bins", t.bins)]) if t.kind == "color_histogram" \
            else _digest("depth_proxy")
        c.const(b"\x00" + struct.pack(">Q", dg))
    c.const(_str8("make_patch") + b"\x00" + _str8(vid))
    c.col(">u8", fno)
    c.const(b"\x01")
    box = np.stack([x1, y1, x2, y2], axis=1) if n else np.zeros((0, 4), np.uint32)
    c.col(">u4", box)
    c.col(">u8", reg_digest)
    c.const(struct.pack(">H", 5 if depth else 4))
    c.const(_str8("bbox") + b"\x03")
    c.col(">u4", box)
    if depth:
        c.const(_str8("depth") + b"\x01")
        c.col(">f8", depth_v)
    c.const(_str8("frame_h") + b"\x00" + struct.pack(">q", H) +
            _str8("frame_w") + b"\x00" + struct.pack(">q", W) + _str8("frameno") + b"\x00")
    c.col(">i8", fno.astype(np.int64))
    rec = c.build(n)
    rec["f0"] = rec.dtype.itemsize - 4
    blob = rec.tobytes()
    R = rec.dtype.itemsize

    # record store: patches, then the collection descriptor and forward index
    fwd = {(vid, f): [int(x) for x in final_ids[f * T:(f + 1) * T]] for f in range(F)} if T else {}
    desc = b"PCOL" + struct.pack(">Q", n)
    fwd_blob = _serialize_forward(fwd)
    try:
        f = open(etl.output, "wb")
    except OSError:
        raise IoError("cannot open record store at " + etl.output)
    with f:
        f.write(_FILE_MAGIC)
        f.write(blob)
        pos = 8 + len(blob)
        f.write(desc)
        f.write(fwd_blob)
        ent = np.empty(n, dtype=np.dtype([("kl", ">u4"), ("key", ">u8"), ("off", ">u8"),
                                          ("len", ">u8")]))
        ent["kl"] = 8
        ent["key"] = final_ids
        ent["off"] = 8 + np.arange(n, dtype=np.uint64) * np.uint64(R)
        ent["len"] = R
        tail = (struct.pack(">I", len(_COLLECTION_KEY)) + _COLLECTION_KEY +
                struct.pack(">QQ", pos, len(desc)) +
                struct.pack(">I", len(_FORWARD_KEY)) + _FORWARD_KEY +
                struct.pack(">QQ", pos + len(desc), len(fwd_blob)))
        f.write(ent.tobytes() + tail)
        f.write(struct.pack(">QQ", pos + len(desc) + len(fwd_blob), n + 2) + _FOOTER_MAGIC)
        size = f.tell()

    # in-memory patches for the executor
    ops = [(t.kind, _digest("color_histogram", [("bins", t.bins)])
            if t.kind == "color_histogram" else _digest("depth_proxy")) for t in chain]
    patches = []
    idl = ids.tolist()
    fl = fno.tolist()
    bl = box.tolist()
    dl = reg_digest.tolist()
    dv = depth_v.tolist() if depth else None
    for i in range(n):
        b = tuple(bl[i])
        meta = {"bbox": b, "frame_h": H, "frame_w": W, "frameno": fl[i]}
        if depth:
            meta["depth"] = dv[i]
        lin = [LineageStep(op, idl[i] + j, None, dg)
               for j, (op, dg) in reversed(list(enumerate(ops)))]
        lin.append(LineageStep("make_patch", (vid, fl[i]), BoundingBox(*b), dl[i]))
        patches.append(Patch(idl[i] + m, data[i], shape, meta, lin))
    return PatchCollection(etl.output, patches, fwd, size, record_bytes=n * R)


# ---------------------------------------------------------------------------
# Predicates (src/query.cpp:30-175)


def _fmt(v: float) -> str:
    return "%g" % v


def _meta_to_string(v) -> str:
    t = _tag(v)
    if t == 0:
        return str(int(v))
    if t == 1:
        return _fmt(v)
    if t == 2:
        return f"'{v}'"
    if t == 3:
        return "[" + ";".join(str(x) for x in _box(v)) + "]"
    return "{" + ";".join(v) + "}"


def _slot(t, slot, what):
    if slot >= len(t):
        raise ConfigError(f"{what} references slot {slot} of a {len(t)}-wide tuple")
    return t[slot]


def _resolve(o: Operand, t):
    if o.slot < 0:
        return o.literal
    p = _slot(t, o.slot, "predicate")
    if "." in o.key:
        base, comp = o.key.split(".", 1)
        v = p.meta.get(base)
        if v is None:
            return None
        if _tag(v) != 3:
            raise TagMismatchError(f"key '{base}' holds {_TAG_NAMES[_tag(v)]}, "
                                   "component access needs a box")
        b = _box(v)
        if comp not in ("x1", "y1", "x2", "y2"):
            raise ConfigError(f"unknown box component '{comp}'")
        return b[("x1", "y1", "x2", "y2").index(comp)]
    return p.meta.get(o.key)


_ORD = {"eq": lambda a, b: a == b, "ne": lambda a, b: a != b, "lt": lambda a, b: a < b,
        "le": lambda a, b: a <= b, "gt": lambda a, b: a > b, "ge": lambda a, b: a >= b}


def _cmp_values(op, l, r, offset) -> bool:
    """eval_cmp_values (src/query.cpp:99-131)."""
    lt, rt = _tag(l), _tag(r)
    if lt <= 1 and rt <= 1:
        return _ORD[op](float(l), float(r) + offset)
    if offset != 0.0:
        raise ConfigError("numeric offset applied to non-numeric operands")
    if lt != rt:
        raise TagMismatchError(f"cannot compare {_TAG_NAMES[lt]} with {_TAG_NAMES[rt]}")
    if lt == 2:
        return _ORD[op](l.encode(), r.encode())
    if op == "eq":
        return _canon(l) == _canon(r)
    if op == "ne":
        return _canon(l) != _canon(r)
    raise TagMismatchError(f"ordering is undefined for {_TAG_NAMES[lt]} values")


def _canon(v):
    t = _tag(v)
    if t == 3:
        return (3, _box(v))
    if t == 4:
        return (4, tuple(v))
    return (t, v)


class _WithinTable:
    """GPU-evaluated ``within`` atoms for one predicate over a tuple list
    (select) or a left x right tuple grid (nl_join).  Each atom's value is
    looked up by (left index, right index); dimension mismatches are kept
    and raised only when the interpreter reaches that atom, as eval_view
    would."""

    def __init__(self):
        self.atoms = {}

    def value(self, atom: Predicate, i: int, j: int) -> bool:
        fn = self.atoms[id(atom)]
        return fn(i, j)


def _data_rows(patches: Sequence[Patch]):
    return [np.asarray(p.data, dtype=np.float32).ravel() for p in patches]


def _rows_within(A: List[np.ndarray], B: List[np.ndarray], radius: float) -> np.ndarray:
    """dist(A[k], B[k]) <= radius for equal-dimension row pairs (GPU)."""
    n = len(A)
    out = np.zeros(n, dtype=np.uint8)
    if n == 0:
        return out.astype(bool)
    dims = np.array([a.size for a in A])
    for d in np.unique(dims):
        idx = np.flatnonzero(dims == d)
        if d == 0:
            out[idx] = radius >= 0
            continue
        Am = np.ascontiguousarray(np.stack([A[k] for k in idx]))
        Bm = np.ascontiguousarray(np.stack([B[k] for k in idx]))
        o = np.empty(len(idx), dtype=np.uint8)
        pdb._check(capi.lib().pdb_rows_within(capi.ptr(Am), capi.ptr(Bm), len(idx), int(d),
                                              float(radius), capi.ptr(o)))
        out[idx] = o
    return out.astype(bool)


def _cross_within(A: List[np.ndarray], B: List[np.ndarray], radius: float):
    """Pairs (i, j), dims equal, dist(A[i], B[j]) <= radius: the GPU join per
    dimension class, sorted in nested-loop order."""
    if not A or not B:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    da = np.array([a.size for a in A])
    db = np.array([b.size for b in B])
    li, ri = [], []
    for d in np.intersect1d(np.unique(da), np.unique(db)):
        ia, ib = np.flatnonzero(da == d), np.flatnonzero(db == d)
        if d == 0:
            if radius >= 0:
                g = np.array(np.meshgrid(ia, ib, indexing="ij")).reshape(2, -1)
                li.append(g[0])
                ri.append(g[1])
            continue
        if radius < 0:
            continue
        Am = np.stack([A[k] for k in ia])
        Bm = np.stack([B[k] for k in ib])
        res = pdb.sim_join(Am, Bm, radius, sort=False)
        li.append(ia[res.left.astype(np.int64)])
        ri.append(ib[res.right.astype(np.int64)])
    if not li:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    a, b = np.concatenate(li), np.concatenate(ri)
    o = np.lexsort((b, a))
    return a[o], b[o]


def _first_mismatch(da: np.ndarray, db: np.ndarray):
    """First (i, j) in nested-loop order with differing dimensions, or None."""
    if da.size == 0 or db.size == 0:
        return None
    ub = np.unique(db)
    if ub.size > 1:
        return 0, int(np.flatnonzero(db != da[0])[0])
    bad = np.flatnonzero(da != ub[0])
    return (int(bad[0]), 0) if bad.size else None


def _within_atoms(p: Predicate, out: list) -> None:
    if p.kind == "within":
        out.append(p)
    for c in p.parts:
        _within_atoms(c, out)


def _mismatch_error(a: Patch, b: Patch):
    return DimensionMismatchError(
        f"distance between {np.asarray(a.data).size} and {np.asarray(b.data).size} "
        "dimensional patches")


def _prepare_within(pred: Predicate, left: List[tuple], right: Optional[List[tuple]],
                    pairs=None, skip: Optional[Predicate] = None):
    """Evaluate every within atom of ``pred`` (but ``skip``) on the GPU.
    Tuples are left[i] (+ right[j] for nl_join); with ``pairs`` = (li, ri)
    only those (i, j) are prepared.  Slots beyond the tuple width are left
    to the interpreter (ConfigError on evaluation)."""
    table = _WithinTable()
    atoms: list = []
    _within_atoms(pred, atoms)
    atoms = [a for a in atoms if a is not skip]
    wl = len(left[0]) if left else 0
    wr = (len(right[0]) if right else 0) if right is not None else 0
    for a in atoms:
        sa, sb = a.slot_a, a.slot_b
        width = wl + wr
        if right is None:
            width = wl
        if sa >= width or sb >= width or not left or (right is not None and not right):
            table.atoms[id(a)] = None
            continue
        side_a = sa >= wl
        side_b = sb >= wl
        if side_a == side_b:
            # both slots in one input: one row pair per tuple of that side
            rows = right if side_a else left
            off = wl if side_a else 0
            pa = [t[sa - off] for t in rows]
            pb = [t[sb - off] for t in rows]
            A, B = _data_rows(pa), _data_rows(pb)
            eq = np.array([x.size == y.size for x, y in zip(A, B)])
            ok = np.zeros(len(rows), dtype=bool)
            if eq.any():
                idx = np.flatnonzero(eq)
                ok[idx] = _rows_within([A[k] for k in idx], [B[k] for k in idx], a.radius)

            def fn(i, j, ok=ok, eq=eq, pa=pa, pb=pb, side=side_a):
                k = j if side else i
                if not eq[k]:
                    raise _mismatch_error(pa[k], pb[k])
                return bool(ok[k])
            table.atoms[id(a)] = fn
            continue
        # cross-side: the left slot against the right slot
        ls, rs = (sa, sb - wl) if not side_a else (sb, sa - wl)
        pl = [t[ls] for t in left]
        pr = [t[rs] for t in right]
        A, B = _data_rows(pl), _data_rows(pr)
        swap = side_a   # euclidean(slot_a, slot_b): report sizes in that order
        if pairs is not None:
            ci, cj = pairs
            lut = {(int(x), int(y)): k for k, (x, y) in enumerate(zip(ci, cj))}
            eq = np.array([A[x].size == B[y].size for x, y in zip(ci, cj)], dtype=bool)
            ok = np.zeros(len(ci), dtype=bool)
            if eq.any():
                idx = np.flatnonzero(eq)
                ok[idx] = _rows_within([A[ci[k]] for k in idx], [B[cj[k]] for k in idx],
                                       a.radius)

            def fn(i, j, lut=lut, eq=eq, ok=ok, pl=pl, pr=pr, swap=swap):
                k = lut[(i, j)]
                if not eq[k]:
                    raise _mismatch_error(pr[j], pl[i]) if swap else \
                        _mismatch_error(pl[i], pr[j])
                return bool(ok[k])
            table.atoms[id(a)] = fn
            continue
        li, ri = _cross_within(A, B, a.radius)
        hit = np.zeros((len(left), len(right)), dtype=bool)
        hit[li, ri] = True
        da = np.array([x.size for x in A])
        db = np.array([x.size for x in B])

        def fn(i, j, hit=hit, da=da, db=db, pl=pl, pr=pr, swap=swap):
            if da[i] != db[j]:
                raise _mismatch_error(pr[j], pl[i]) if swap else _mismatch_error(pl[i], pr[j])
            return bool(hit[i, j])
        table.atoms[id(a)] = fn
    return table


def _eval(p: Predicate, t, table: _WithinTable, i: int, j: int) -> bool:
    """eval_view (src/query.cpp:133-175) with within atoms from the GPU."""
    k = p.kind
    if k == "cmp":
        lv = _resolve(p.lhs, t)
        if lv is None:
            return False
        rv = _resolve(p.rhs, t)
        if rv is None:
            return False
        return _cmp_values(p.op, lv, rv, p.offset)
    if k == "within":
        a = _slot(t, p.slot_a, "distance predicate")
        b = _slot(t, p.slot_b, "distance predicate")
        fn = table.atoms.get(id(p))
        if fn is None:  # unreachable: prepared for every in-range atom
            raise Error("within atom was not prepared")
        del a, b
        return fn(i, j)
    if k == "contains":
        a = _slot(t, p.slot_a, "contains predicate")
        v = a.meta.get(p.key)
        if v is None:
            return False
        if _tag(v) != 4:
            raise TagMismatchError(f"key '{p.key}' holds {_TAG_NAMES[_tag(v)]}, "
                                   "contains needs a string list")
        return p.needle in v
    if k == "and":
        return all(_eval(c, t, table, i, j) for c in p.parts)
    if k == "or":
        return any(_eval(c, t, table, i, j) for c in p.parts)
    if len(p.parts) != 1:
        raise ConfigError("negation takes exactly one child predicate")
    return not _eval(p.parts[0], t, table, i, j)


# ---------------------------------------------------------------------------
# Executor (src/query.cpp:584-1029)


@dataclass
class _OpStats:
    label: str
    ms: float = 0.0
    tuples_out: int = 0
    index_probes: int = 0


class _Executor:
    def __init__(self, collections: Dict[str, PatchCollection]):
        self.cols = collections
        self.ops: List[_OpStats] = []
        self.records_read = 0
        self.bytes_read = 0

    def number(self, n: PlanNode) -> None:
        """Compiler::compile's pre-order operator numbering."""
        n.op_index = len(self.ops)
        self.ops.append(_OpStats(n.label()))
        if n.kind == "scan" and n.collection not in self.cols:
            raise ConfigError(f"collection '{n.collection}' is not registered")
        for c in n.children:
            self.number(c)

    def run(self, n: PlanNode) -> List[tuple]:
        t0 = time.perf_counter()
        out = getattr(self, "_" + n.kind)(n)
        st = self.ops[n.op_index]
        st.ms += (time.perf_counter() - t0) * 1e3
        st.tuples_out += len(out)
        return out

    def _scan(self, n):
        col = self.cols[n.collection]
        self.records_read += len(col.patches)
        self.bytes_read += col.record_bytes
        return [(p,) for p in col.patches]

    def _select(self, n):
        rows = self.run(n.children[0])
        table = _prepare_within(n.pred, rows, None)
        return [t for i, t in enumerate(rows) if _eval(n.pred, t, table, i, i)]

    def _nl_join(self, n):
        right = self.run(n.children[1])     # drained before the first left pull
        left = self.run(n.children[0])
        if not left or not right:
            return []
        pred = n.pred
        wl = len(left[0])
        lead = pred if pred.kind == "within" else (
            pred.parts[0] if pred.kind == "and" and pred.parts and
            pred.parts[0].kind == "within" else None)
        if lead is not None and (lead.slot_a < wl) != (lead.slot_b < wl) and \
                max(lead.slot_a, lead.slot_b) < wl + len(right[0]):
            # the join's candidates come from the GPU join of the lead atom
            sa, sb = lead.slot_a, lead.slot_b
            ls, rs = (sa, sb - wl) if sa < wl else (sb, sa - wl)
            A = _data_rows([t[ls] for t in left])
            B = _data_rows([t[rs] for t in right])
            mm = _first_mismatch(np.array([x.size for x in A]), np.array([x.size for x in B]))
            li, ri = _cross_within(A, B, lead.radius)
            if mm is not None:
                # the first mismatched pair in loop order raises; candidates
                # before it are evaluated first (their outputs are discarded)
                i, j = mm
                before = (li < i) | ((li == i) & (ri < j))
                li, ri = li[before], ri[before]
            rest = pred.parts[1:] if pred.kind == "and" else []
            table = _prepare_within(pred, left, right, (li, ri), skip=lead) if rest else None
            out = []
            for a, b in zip(li.tolist(), ri.tolist()):
                t = left[a] + right[b]
                if all(_eval(c, t, table, a, b) for c in rest):
                    out.append(t)
            if mm is not None:
                t = left[mm[0]] + right[mm[1]]
                raise _mismatch_error(t[lead.slot_a], t[lead.slot_b])
            return out
        table = _prepare_within(pred, left, right)
        out = []
        for a, lt in enumerate(left):
            for b, rt in enumerate(right):
                t = lt + rt
                if _eval(pred, t, table, a, b):
                    out.append(t)
        return out

    @staticmethod
    def _singles(rows, what):
        for t in rows:
            if len(t) != 1:
                raise ValidationError(f"{what} operates on single-patch tuples, got width "
                                      f"{len(t)}")
        return [t[0] for t in rows]

    def _sim_join(self, n):
        L = self._singles(self.run(n.children[0]), "similarity join")
        R = self._singles(self.run(n.children[1]), "similarity join")
        probes: list = []
        pairs = pdb.sim_join_pairs(L, R, n.tau, n.side, probes)
        self.ops[n.op_index].index_probes += probes[0] if probes else 0
        return [(a, b) for a, b in pairs]

    def _dedup(self, n):
        items = self._singles(self.run(n.children[0]), "dedup")
        return [(p,) for p in pdb.dedup_groups(items, n.tau)]

    def _count_by(self, n):
        items = self._singles(self.run(n.children[0]), "count_by")
        groups: Dict[object, list] = {}
        order = []
        for p in items:
            v = p.meta.get(n.key)
            if v is None:
                continue
            k = _canon(v)
            if k in groups:
                groups[k][1] += 1
            else:
                groups[k] = [p, 1]
                order.append(k)
        dg = _digest("count_by", [("key", n.key)])
        out = []
        for k in order:
            first, cnt = groups[k]
            meta = dict(first.meta)
            meta["count"] = cnt
            out.append((Patch(pdb.next_patch_id(), first.data, tuple(first.shape), meta,
                              [LineageStep("count_by", first.patch_id, None, dg)] +
                              list(first.lineage)),))
        return out


def _stats_text(ops: List[_OpStats], n_tuples: int, total_ms: float, records_read: int,
                bytes_read: int) -> str:
    """ExecStats::to_text (src/query.cpp:1031-1045)."""
    s = f"{len(ops)} operators; {n_tuples} tuples; {_fmt(total_ms)} ms total\n"
    for o in ops:
        s += f"  {o.label}: tuples_out={o.tuples_out} ms={_fmt(o.ms)}"
        if o.index_probes:
            s += f" probes={o.index_probes}"
        s += "\n"
    return s + f"io: records_read={records_read} bytes_read={bytes_read} frames_decoded=0\n"


def _stats_csv(ops: List[_OpStats], n_tuples: int, total_ms: float) -> str:
    """ExecStats::to_csv (src/query.cpp:1047-1058)."""
    s = "op,ms,tuples_out,index_probes\n"
    probes = 0
    for o in ops:
        s += f"{o.label},{_fmt(o.ms)},{o.tuples_out},{o.index_probes}\n"
        probes += o.index_probes
    return s + f"total,{_fmt(total_ms)},{n_tuples},{probes}\n"


def _meta_py(v):
    t = _tag(v)
    if t == 3:
        return _box(v)
    if t == 4:
        return list(v)
    return v


def patch_to_py(p: Patch, with_data: bool = False, with_lineage: bool = False) -> dict:
    """patch_to_py (bindings/py_module.cpp:20-29); ``with_lineage`` adds the
    lineage steps (op, frame | parent, digest, region) for parity checks."""
    d = {"id": int(p.patch_id), "shape": [int(x) for x in p.shape],
         "meta": {k: _meta_py(p.meta[k]) for k in _meta_keys(p.meta)}}
    if with_data:
        d["data"] = np.asarray(p.data, dtype=np.float32).ravel().tolist()
    if with_lineage:
        lin = []
        for st in p.lineage:
            e = {"op": st.op_name, "digest": int(st.params_digest)}
            if isinstance(st.source, tuple):
                e["frame"] = [st.source[0], int(st.source[1])]
            else:
                e["parent"] = int(st.source)
            if st.region is not None:
                e["region"] = list(_box(st.region))
            lin.append(e)
        d["lineage"] = lin
    return d


# ---------------------------------------------------------------------------
# Entry points (bindings/py_module.cpp)


def run_etl(plan_json: str) -> dict:
    """run_etl (bindings/py_module.cpp:139-166)."""
    pf = parse_plan(plan_json)
    if pf.etl is None:
        raise ValidationError("plan file has no etl section")
    check_stages(pf)
    if pf.index_builds:
        raise UnsupportedError("indexes: secondary indexes are outside the B200 build's scope")
    col = materialize_etl(pf)
    return {"patches": col.patch_count(), "output": col.path(), "indexes": []}


def run_query(plan_json: str, with_data: bool = False, with_lineage: bool = False) -> dict:
    """run_query (bindings/py_module.cpp:168-213)."""
    pf = parse_plan(plan_json)
    if pf.plan is None:
        raise ValidationError("plan file has no plan section")
    check_stages(pf)
    cols: Dict[str, PatchCollection] = {}
    if pf.etl is not None:
        cols[pf.etl.name] = materialize_etl(pf)
    for alias, path in pf.collections.items():
        if alias not in cols:
            cols[alias] = PatchCollection.open(path)
    for alias, path in pf.stores.items():
        pdb.VideoStore.open(path).close()
    if pf.load_indexes:
        raise UnsupportedError("load_indexes: secondary indexes are outside the B200 build's "
                               "scope")
    ex = _Executor(cols)
    ex.number(pf.plan)
    t0 = time.perf_counter()
    tuples = ex.run(pf.plan)
    total = (time.perf_counter() - t0) * 1e3
    return {
        "tuples": [[patch_to_py(p, with_data, with_lineage) for p in t] for t in tuples],
        "traced": [],
        "stats_text": _stats_text(ex.ops, len(tuples), total, ex.records_read, ex.bytes_read),
        "stats_csv": _stats_csv(ex.ops, len(tuples), total),
        "records_read": ex.records_read,
        "frames_decoded": 0,
    }


def collection_patches(path: str, with_data: bool = False) -> list:
    """collection_patches (bindings/py_module.cpp:322-331)."""
    return [patch_to_py(p, with_data) for p in PatchCollection.open(path).patches]


def collection_stats(path: str) -> dict:
    """collection_stats (bindings/py_module.cpp:308-320)."""
    col = PatchCollection.open(path)
    return {"patches": col.patch_count(), "frames_covered": len(col.fwd), "bytes": col.size,
            "indexes": col.index_names}


_LAYOUTS = ("frame_file", "encoded_file", "segmented_file")
_QUALITY = {4: "high", 16: "medium", 64: "low"}


def store_stats(path: str) -> dict:
    """store_stats (bindings/py_module.cpp:291-306)."""
    vs = pdb.VideoStore.open(path)
    try:
        i = vs.info
        return {"video_id": vs.video_id, "frames": vs.frame_count, "width": vs.width,
                "height": vs.height, "layout": _LAYOUTS[i.layout],
                "quality": "none" if i.codec_mode == 0 else _QUALITY.get(i.quant_step, "?"),
                "clip_len": int(i.clip_len), "bytes": os.path.getsize(path)}
    finally:
        vs.close()

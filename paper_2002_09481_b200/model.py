"""Model files and the Conv2D -> AxConv2D ``transform``.

Graphs are lists of node dicts ``{"id", "kind", "inputs", "attrs"}`` in the
reference's vocabulary (``axemu.graph.NodeKind``, graph.py:25-37), the form
``GpuGraph`` executes.  This module restates, with the same semantics and
diagnostics:

* ``validate``      <- ``LayerGraph.validate`` (graph.py:55-83)
* ``transform``     <- ``transform`` (graph.py:107-141): every Conv2D becomes an
  AxConv2D fed by fresh ``<id>.in_min`` / ``<id>.in_max`` batch range nodes,
  with the filter range folded to constants ``f_min`` / ``f_max``;
* ``save_model`` / ``load_model`` <- formats.py:298-377: a JSON document plus a
  little-endian float32 weight sidecar, truth tables as sibling ``.axm`` files
  (byte-identical documents and sidecars for the same graph).

So a model file written by the reference loads here and runs on the GPU:
``GpuGraph(load_model("net.json"))``.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .formats import FormatError, load_lut, save_lut
from .types import MultLut

MODEL_FORMAT = "axemu-model"
NODE_KINDS = ("Input", "Conv2D", "AxConv2D", "Min", "Max", "ReLU", "MaxPool", "AvgPool", "Add", "Dense",
              "Flatten", "Softmax")


def node(nid: str, kind: str, inputs=(), **attrs) -> dict:
    return {"id": nid, "kind": kind, "inputs": list(inputs), "attrs": dict(attrs)}


def _kind(n: dict) -> str:
    k = n["kind"]
    return getattr(k, "value", k)


def validate(nodes: list[dict]) -> None:
    """graph.py:55-83: ids unique and non-empty, inputs precede, constant weights, AxConv2D arity."""
    seen: set[str] = set()
    for n in nodes:
        nid, kind = n["id"], _kind(n)
        if not nid:
            raise ValueError("node id must be non-empty")
        if nid in seen:
            raise ValueError(f"duplicate node id {nid!r}")
        if kind not in NODE_KINDS:
            raise ValueError(f"unknown node kind {kind!r}")
        for ref in n.get("inputs", []):
            if ref not in seen:
                raise ValueError(f"node {nid!r} references {ref!r} which does not precede it")
        attrs = n.get("attrs", {})
        if kind == "Conv2D" and not isinstance(attrs.get("filters"), np.ndarray):
            raise ValueError(f"Conv2D node {nid!r} has no constant filters")
        if kind == "Dense" and not isinstance(attrs.get("weights"), np.ndarray):
            raise ValueError(f"Dense node {nid!r} has no constant weights")
        if kind == "AxConv2D":
            if len(n.get("inputs", [])) != 3:
                raise ValueError(f"AxConv2D node {nid!r} needs data, min, and max inputs")
            for key in ("filters", "lut", "f_min", "f_max"):
                if key not in attrs:
                    raise ValueError(f"AxConv2D node {nid!r} missing {key!r}")
        seen.add(nid)


@dataclass(frozen=True)
class TransformReport:
    replaced_count: int
    inserted_min_max: int
    untouched_kinds: list


def transform(nodes: list[dict], lut: MultLut) -> tuple[list[dict], TransformReport]:
    """Replace every Conv2D by AxConv2D fed by fresh batch Min/Max range nodes (graph.py:107-141)."""
    validate(nodes)
    existing = {n["id"] for n in nodes}
    out: list[dict] = []
    replaced = 0
    untouched: set[str] = set()
    for n in nodes:
        kind = _kind(n)
        if kind != "Conv2D":
            untouched.add(kind)
            out.append(n)
            continue
        filters = n["attrs"].get("filters")
        if not isinstance(filters, np.ndarray):
            raise ValueError(f"Conv2D node {n['id']!r} has non-constant filters")
        data_id = n["inputs"][0]
        min_id, max_id = f"{n['id']}.in_min", f"{n['id']}.in_max"
        if min_id in existing or max_id in existing:
            raise ValueError(f"range node ids for {n['id']!r} already taken")
        existing.update((min_id, max_id))
        out.append(node(min_id, "Min", [data_id]))
        out.append(node(max_id, "Max", [data_id]))
        attrs = dict(n["attrs"])
        attrs["f_min"] = float(filters.min())
        attrs["f_max"] = float(filters.max())
        attrs["lut"] = lut
        out.append(node(n["id"], "AxConv2D", [data_id, min_id, max_id], **attrs))
        replaced += 1
    validate(out)
    return out, TransformReport(replaced, 2 * replaced, sorted(untouched))


# ---------------------------------------------------------------------------- model files


def _encode_attr(value, blobs: list, luts: list):
    if isinstance(value, np.ndarray):
        offset = sum(b.size for b in blobs)
        blobs.append(np.ascontiguousarray(value, dtype=np.float32))
        return {"__blob__": {"offset": offset, "shape": list(value.shape)}}
    if isinstance(value, MultLut) or (hasattr(value, "mode") and hasattr(value, "entries")):
        for i, existing in enumerate(luts):
            if existing is value:
                return {"__lut__": i}
        luts.append(value)
        return {"__lut__": len(luts) - 1}
    if isinstance(value, tuple):
        return list(value)
    return value


def _decode_attr(value, weights: np.ndarray, luts: list):
    if isinstance(value, dict) and "__blob__" in value:
        ref = value["__blob__"]
        shape = tuple(ref["shape"])
        count = int(np.prod(shape)) if shape else 1
        start = int(ref["offset"])
        return weights[start:start + count].reshape(shape).copy()
    if isinstance(value, dict) and "__lut__" in value:
        return luts[int(value["__lut__"])]
    return value


def save_model(nodes: list[dict], path: str | Path, lut_path: str | Path | None = None) -> None:
    """Model JSON plus a float32 weight sidecar next to it (formats.py:298-339)."""
    path = Path(path)
    blobs: list[np.ndarray] = []
    luts: list = []
    nodes_doc = []
    for n in nodes:
        attrs_doc = {k: _encode_attr(v, blobs, luts) for k, v in n.get("attrs", {}).items()}
        nodes_doc.append({"id": n["id"], "kind": _kind(n), "inputs": list(n.get("inputs", [])), "attrs": attrs_doc})
    lut_names = []
    for i, lut in enumerate(luts):
        if lut_path is not None and i == 0:
            name = str(lut_path)
        else:
            name = path.stem + (f".{i}" if i else "") + ".axm"
            save_lut(lut, path.parent / name)
        lut_names.append(name)
    weights_name = path.stem + ".weights.bin"
    doc = {"format": MODEL_FORMAT, "version": 1, "weights_file": weights_name, "luts": lut_names,
           "nodes": nodes_doc}
    blob = np.concatenate([b.ravel() for b in blobs]) if blobs else np.empty(0, dtype=np.float32)
    (path.parent / weights_name).write_bytes(blob.astype("<f4").tobytes())
    path.write_text(json.dumps(doc, indent=1) + "\n")


def load_model(path: str | Path) -> list[dict]:
    """formats.py:342-377; returns validated node dicts."""
    path = Path(path)
    try:
        doc = json.loads(path.read_text())
    except json.JSONDecodeError as e:
        raise FormatError(f"malformed model document: {e}") from e
    if doc.get("format") != MODEL_FORMAT:
        raise FormatError(f"not a model file (format={doc.get('format')!r})")
    weights = np.frombuffer((path.parent / doc["weights_file"]).read_bytes(), dtype="<f4")
    luts = [load_lut(path.parent / name) for name in doc.get("luts", [])]
    nodes = []
    for nd in doc["nodes"]:
        if nd["kind"] not in NODE_KINDS:
            raise FormatError(f"unknown node kind {nd['kind']!r} in {nd['id']!r}")
        attrs = {k: _decode_attr(v, weights, luts) for k, v in nd["attrs"].items()}
        nodes.append(node(nd["id"], nd["kind"], nd["inputs"], **attrs))
    validate(nodes)
    return nodes

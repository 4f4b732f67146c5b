"""Model description consumed by the runtime: parameters, operators, AC groups.

This is the host-side input of the chunk store. It carries the same records
as the reference profile (offplan/profiles.py:53-223) so a plan produced by
the reference planner for a profile applies unchanged to a model described
here, and offplan objects can be passed wherever these are accepted (every
function below reads attributes only).

Provided here:
  * PrecisionSpec           — byte widths (profiles.py:53-76)
  * ParameterSpec / OperatorNode / ModelProfile / AccessTrace
  * synthesize_transformer_profile — GPT-2 records in forward order
                              (profiles.py:408-482)
  * coarsen_graph           — AC-group merge (profiles.py:490-521)
  * partition_multiuse      — shared split + first-use order (chunking.py:82-99)
  * JSON load/dump of the model-profile format (profiles.py:268-339)
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Any, Iterable, Sequence

from .errors import ProfileFormatError, UncommonGraphError, ValidationError

FORMAT_VERSION = 1


@dataclass(frozen=True)
class PrecisionSpec:
    """Per-element widths: compute (L_c), optimizer (L_os), optimizer factor (F_os)."""

    compute_bytes: int = 2
    optimizer_bytes: int = 4
    optimizer_factor: int = 3

    def __post_init__(self) -> None:
        if min(self.compute_bytes, self.optimizer_bytes, self.optimizer_factor) <= 0:
            raise ValidationError("precision widths must be strictly positive")

    @property
    def optimizer_state_bytes(self) -> int:
        return self.optimizer_bytes * self.optimizer_factor


@dataclass(frozen=True)
class ParameterSpec:
    id: str
    numel: int
    shared: bool = False

    def __post_init__(self) -> None:
        if not self.id:
            raise ValidationError("parameter id must be non-empty")
        if self.numel < 1:
            raise ValidationError(f"parameter '{self.id}': numel must be >= 1")


@dataclass(frozen=True)
class OperatorNode:
    name: str
    param_ids: tuple[str, ...]
    ac_group: int | None = None


@dataclass(frozen=True)
class ModelProfile:
    name: str
    parameters: tuple[ParameterSpec, ...]
    operators: tuple[OperatorNode, ...]
    activation_bytes: int = 0
    buffer_bytes: int = 0

    def __post_init__(self) -> None:
        ids = [p.id for p in self.parameters]
        if len(set(ids)) != len(ids):
            dup = next(i for i in ids if ids.count(i) > 1)
            raise ValidationError(f"duplicate parameter id '{dup}'")
        known = set(ids)
        read: set[str] = set()
        for op in self.operators:
            for pid in op.param_ids:
                if pid not in known:
                    raise ValidationError(f"operator '{op.name}' references unknown parameter '{pid}'")
                read.add(pid)
        for p in self.parameters:
            if not p.shared and p.id not in read:
                raise ValidationError(f"parameter '{p.id}' is not read by any operator")

    def numel_of(self, pid: str) -> int:
        for p in self.parameters:
            if p.id == pid:
                return p.numel
        raise ValidationError(f"unknown parameter id '{pid}'")

    @property
    def total_elements(self) -> int:
        return sum(p.numel for p in self.parameters)


@dataclass(frozen=True)
class AccessTrace:
    coarse_ops: tuple[frozenset[str], ...]
    shared_param_ids: frozenset[str] = field(default_factory=frozenset)


# --------------------------------------------------------------------------
# GPT-2 records (forward order) — the layout every plan for this model uses.
# --------------------------------------------------------------------------

# Per-layer tensors as (suffix, numel(h)) in forward order; each layer is one
# AC group of six operators (profiles.py:447-463).
_LAYER_OPS = (
    ("ln_1", (("ln_1.w", lambda h: h), ("ln_1.b", lambda h: h))),
    ("attn.qkv", (("attn.qkv.w", lambda h: 3 * h * h), ("attn.qkv.b", lambda h: 3 * h))),
    ("attn.proj", (("attn.proj.w", lambda h: h * h), ("attn.proj.b", lambda h: h))),
    ("ln_2", (("ln_2.w", lambda h: h), ("ln_2.b", lambda h: h))),
    ("mlp.fc", (("mlp.fc.w", lambda h: 4 * h * h), ("mlp.fc.b", lambda h: 4 * h))),
    ("mlp.proj", (("mlp.proj.w", lambda h: 4 * h * h), ("mlp.proj.b", lambda h: h))),
)


def synthesize_transformer_profile(hidden: int, layers: int, heads: int, vocab: int,
                                   seq_len: int, batch: int, name: str | None = None) -> ModelProfile:
    """GPT-2 decoder records: tied wte (shared), wpe, L AC-grouped layers, ln_f, lm_head."""
    for label, val in (("hidden", hidden), ("layers", layers), ("heads", heads),
                       ("vocab", vocab), ("seq_len", seq_len), ("batch", batch)):
        if val < 1:
            raise ValidationError(f"{label} must be >= 1")
    h = hidden
    params = [ParameterSpec("wte", vocab * h, shared=True), ParameterSpec("wpe", seq_len * h)]
    ops = [OperatorNode("embed", ("wte", "wpe"))]
    for i in range(layers):
        for op_name, tensors in _LAYER_OPS:
            ids = []
            for suffix, size in tensors:
                pid = f"h{i}.{suffix}"
                params.append(ParameterSpec(pid, size(h)))
                ids.append(pid)
            ops.append(OperatorNode(f"h{i}.{op_name}", tuple(ids), ac_group=i))
    params += [ParameterSpec("ln_f.w", h), ParameterSpec("ln_f.b", h)]
    ops += [OperatorNode("ln_f", ("ln_f.w", "ln_f.b")), OperatorNode("lm_head", ("wte",))]
    # Activation / buffer estimates of the reference generator (profiles.py:472-481).
    activation = 2 * batch * seq_len * hidden * layers * 2
    return ModelProfile(name or f"transformer-h{hidden}-l{layers}", tuple(params), tuple(ops),
                        activation, 2 * seq_len * seq_len)


def coarsen_graph(profile: Any) -> AccessTrace:
    """One coarse node per AC group (at the group's first operator) or per bare
    operator; shared parameters removed (profiles.py:490-521)."""
    shared = frozenset(p.id for p in profile.parameters if p.shared)
    nodes: list[set[str]] = []
    slot_of_group: dict[int, int] = {}
    for op in profile.operators:
        if op.ac_group is None:
            nodes.append(set(op.param_ids))
        elif op.ac_group in slot_of_group:
            nodes[slot_of_group[op.ac_group]].update(op.param_ids)
        else:
            slot_of_group[op.ac_group] = len(nodes)
            nodes.append(set(op.param_ids))
    seen: set[str] = set()
    coarse = []
    for node in nodes:
        kept = frozenset(node) - shared
        clash = kept & seen
        if clash:
            raise UncommonGraphError(
                f"parameter '{min(clash)}' is read by multiple coarse operators; "
                "mark it shared=true or enclose its operators in one ac_group")
        seen |= kept
        coarse.append(kept)
    return AccessTrace(tuple(coarse), shared)


def partition_multiuse(profile: Any) -> tuple[int, tuple[Any, ...]]:
    """(shared element count, single-use parameters sorted by (first use, declaration))."""
    first: dict[str, int] = {}
    for k, op in enumerate(profile.operators):
        for pid in op.param_ids:
            if pid not in first:
                first[pid] = k
    shared_elems = 0
    keyed = []
    for decl, p in enumerate(profile.parameters):
        if p.shared:
            shared_elems += p.numel
        else:
            keyed.append(((first[p.id], decl), p))
    keyed.sort(key=lambda kp: kp[0])
    return shared_elems, tuple(p for _, p in keyed)


# --------------------------------------------------------------------------
# JSON (format_version 1, same schema as profiles.py:14-23)
# --------------------------------------------------------------------------

def load_model_profile(text: str) -> ModelProfile:
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise ProfileFormatError(f"model profile: not valid JSON ({exc})") from None
    if not isinstance(doc, dict) or doc.get("format_version") != FORMAT_VERSION:
        raise ProfileFormatError("model profile: format_version: expected 1")
    try:
        params = tuple(ParameterSpec(str(p["id"]), int(p["numel"]), bool(p["shared"]))
                       for p in doc["parameters"])
        ops = tuple(OperatorNode(str(o["name"]), tuple(o["param_ids"]), o["ac_group"])
                    for o in doc["operators"])
        return ModelProfile(doc["name"], params, ops, int(doc["activation_bytes"]),
                            int(doc["buffer_bytes"]))
    except (KeyError, TypeError) as exc:
        raise ProfileFormatError(f"model profile: malformed field ({exc})") from None


def dump_model_profile(profile: Any) -> str:
    return json.dumps({
        "format_version": FORMAT_VERSION,
        "name": profile.name,
        "parameters": [{"id": p.id, "numel": p.numel, "shared": p.shared} for p in profile.parameters],
        "operators": [{"name": o.name, "param_ids": list(o.param_ids), "ac_group": o.ac_group}
                      for o in profile.operators],
        "activation_bytes": profile.activation_bytes,
        "buffer_bytes": profile.buffer_bytes,
    }, indent=1)


def profile_from_records(name: str, params: Iterable[tuple[str, int, bool]],
                         ops: Sequence[tuple[str, Sequence[str], int | None]]) -> ModelProfile:
    """Build a profile from a live model's records (the pre-runtime profiler output)."""
    return ModelProfile(name, tuple(ParameterSpec(i, n, s) for i, n, s in params),
                        tuple(OperatorNode(a, tuple(b), c) for a, b, c in ops))

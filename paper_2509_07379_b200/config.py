"""Model / cost / policy configuration — the drop-in mirror of the reference's
``duoserve.config`` (``/root/reference/pkg/src/duoserve/config.py``).

Same names, same JSON schema, same validation messages' intent and the same
exception type (``ConfigError(ValueError)``), so callers written against the
reference load presets and size the expert cache identically:

* ``ModelConfig``      — config.py:21-59 (uniform per-expert bytes, :117-120)
* ``CostModel``        — config.py:62-85 (kept for schema parity; real B200
                         timing replaces the simulated cost on the hot path)
* ``SchedulerPolicy``  — config.py:88-98
* ``slot_count``       — config.py:101-114 (ondemand k, duoserve/oracle 2k,
                         prefetchall 2M)
* ``load_config`` / ``save_config`` / ``config_to_json`` / ``load_preset`` /
  ``preset_names``     — config.py:123-205

B200 addition (not in the reference, whose ``ModelConfig`` carries only L/M/k
and byte budgets): ``ModelShape`` — the tensor shapes of the Mixtral-style W4
model the runtime actually executes (hidden size, FFN width, heads, vocab, AWQ
group).  Shapes live in ``shapes/*.json`` so the reference's strict preset
schema is untouched.
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass, fields
from enum import Enum
from pathlib import Path

_HERE = Path(__file__).resolve().parent


class ConfigError(ValueError):
    """Malformed configuration file or violated configuration invariant."""


def derive_expert_bytes(cfg: "ModelConfig") -> int:
    """Per-expert bytes implied by the totals: floor((total - non_moe) / (L*M)).

    Mirrors config.py:117-120 (integer floor division)."""
    return (cfg.total_param_bytes - cfg.non_moe_bytes) // (cfg.num_layers * cfg.num_experts)


@dataclass(frozen=True)
class ModelConfig:
    name: str
    num_layers: int
    num_experts: int
    top_k: int
    total_param_bytes: int
    non_moe_bytes: int
    predictor_mem_bytes: int
    kv_reserve_bytes: int

    def __post_init__(self):
        # invariant checks in the order of config.py:34-55
        L, M, k = self.num_layers, self.num_experts, self.top_k
        if L < 1:
            raise ConfigError(f"num_layers must be >= 1, got {L}")
        if M < 2:
            raise ConfigError(f"num_experts must be >= 2, got {M}")
        if not (1 <= k < M):
            raise ConfigError(f"top_k must satisfy 1 <= top_k < num_experts, got top_k={k}, num_experts={M}")
        if self.non_moe_bytes >= self.total_param_bytes:
            raise ConfigError(
                f"non_moe_bytes ({self.non_moe_bytes}) must be smaller than "
                f"total_param_bytes ({self.total_param_bytes})")
        for name in ("total_param_bytes", "non_moe_bytes", "predictor_mem_bytes", "kv_reserve_bytes"):
            if getattr(self, name) < 0:
                raise ConfigError(f"{name} must be non-negative")
        if self.expert_bytes <= 0:
            raise ConfigError(f"derived expert size must be positive, got {self.expert_bytes}")

    @property
    def expert_bytes(self) -> int:
        return derive_expert_bytes(self)


@dataclass(frozen=True)
class CostModel:
    """Simulated link/compute timing (config.py:62-85).  Only the CPU
    simulator oracle and the calibrated-preset report use it; the B200 runtime
    is timed for real."""

    link_bandwidth_bytes_per_s: float
    link_latency_s: float
    expert_compute_base_s: float
    expert_compute_per_token_s: float
    non_moe_compute_per_layer_s: float
    gate_compute_s: float
    predictor_latency_s: float

    def __post_init__(self):
        for f in fields(self):
            v = getattr(self, f.name)
            if not v > 0:
                raise ConfigError(f"cost model field {f.name} must be strictly positive, got {v}")

    def transfer_time_s(self, nbytes: int) -> float:
        return self.link_latency_s + nbytes / self.link_bandwidth_bytes_per_s


class SchedulerPolicy(str, Enum):
    ON_DEMAND = "ondemand"
    PREFETCH_ALL = "prefetchall"
    DUOSERVE = "duoserve"
    DUOSERVE_ORACLE = "oracle"

    @property
    def needs_predictor(self) -> bool:
        return self is SchedulerPolicy.DUOSERVE


def slot_count(policy: SchedulerPolicy, cfg: ModelConfig) -> int:
    """Device expert-cache capacity per policy (config.py:101-114)."""
    table = {
        SchedulerPolicy.ON_DEMAND: cfg.top_k,
        SchedulerPolicy.DUOSERVE: 2 * cfg.top_k,
        SchedulerPolicy.DUOSERVE_ORACLE: 2 * cfg.top_k,
        SchedulerPolicy.PREFETCH_ALL: 2 * cfg.num_experts,
    }
    try:
        return table[SchedulerPolicy(policy)]
    except (ValueError, KeyError):
        raise ConfigError(f"unknown policy {policy!r}") from None


# --------------------------------------------------------------------------
# JSON I/O (config.py:123-205)

_MODEL_KEYS = tuple(f.name for f in fields(ModelConfig))
_COST_KEYS = tuple(f.name for f in fields(CostModel))
_INT_KEYS = {"num_layers", "num_experts", "top_k", "total_param_bytes", "non_moe_bytes",
             "predictor_mem_bytes", "kv_reserve_bytes"}


def _read_section(doc: dict, key: str, names, path) -> dict:
    sec = doc.get(key)
    if not isinstance(sec, dict):
        raise ConfigError(f"{path}: missing '{key}' section")
    extra = sorted(set(sec) - set(names))
    if extra:
        raise ConfigError(f"{path}: unknown {key} fields {extra}")
    absent = sorted(set(names) - set(sec))
    if absent:
        raise ConfigError(f"{path}: missing {key} fields {absent}")
    out = {}
    for n in names:
        v = sec[n]
        if n == "name":
            if not (isinstance(v, str) and v):
                raise ConfigError(f"{path}: model.name must be a non-empty string")
        elif n in _INT_KEYS:
            if isinstance(v, bool) or not isinstance(v, int):
                raise ConfigError(f"{path}: {key}.{n} must be an integer, got {v!r}")
        else:
            if isinstance(v, bool) or not isinstance(v, (int, float)):
                raise ConfigError(f"{path}: {key}.{n} must be a number, got {v!r}")
            v = float(v)
        out[n] = v
    return out


def load_config(path) -> tuple[ModelConfig, CostModel]:
    path = Path(path)
    try:
        text = path.read_text(encoding="utf-8")
    except OSError as e:
        raise ConfigError(f"cannot read config {path}: {e}") from e
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise ConfigError(f"{path}: line {e.lineno}, column {e.colno}: {e.msg}") from e
    if not isinstance(doc, dict):
        raise ConfigError(f"{path}: top level must be a JSON object")
    return (ModelConfig(**_read_section(doc, "model", _MODEL_KEYS, path)),
            CostModel(**_read_section(doc, "cost", _COST_KEYS, path)))


def config_to_json(cfg: ModelConfig, cost: CostModel) -> str:
    return json.dumps({"model": asdict(cfg), "cost": asdict(cost)}, indent=2, sort_keys=True) + "\n"


def save_config(cfg: ModelConfig, cost: CostModel, path) -> None:
    Path(path).write_text(config_to_json(cfg, cost), encoding="utf-8")


def preset_names() -> list[str]:
    return sorted(p.stem for p in (_HERE / "presets").glob("*.json"))


def load_preset(name: str) -> tuple[ModelConfig, CostModel]:
    p = _HERE / "presets" / f"{name}.json"
    if not p.is_file():
        raise ConfigError(f"unknown preset {name!r}; available: {preset_names()}")
    return load_config(p)


# --------------------------------------------------------------------------
# B200 runtime shapes (not in the reference)

@dataclass(frozen=True)
class ModelShape:
    """Tensor shapes of the executed Mixtral-style model.

    Defaults follow the public Mixtral configs (HF ``MixtralConfig`` defaults
    for 8x7B: d=4096, ff=14336, 32 q / 8 kv heads x 128, vocab 32000)."""

    name: str
    num_layers: int
    num_experts: int
    top_k: int
    hidden: int
    ffn: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    vocab: int
    group_size: int = 128
    rope_theta: float = 1e6
    rms_eps: float = 1e-5

    def __post_init__(self):
        if self.hidden % self.group_size or self.ffn % self.group_size:
            raise ConfigError("hidden and ffn must be multiples of group_size")
        if self.hidden % 128 or self.ffn % 128:
            raise ConfigError("hidden and ffn must be multiples of 128 (kernel tiling)")
        if self.n_heads % self.n_kv_heads:
            raise ConfigError("n_heads must be a multiple of n_kv_heads")
        if not 1 <= self.top_k < self.num_experts <= 64:
            raise ConfigError("need 1 <= top_k < num_experts <= 64")

    # W4 (AWQ-style, group G) expert: three matrices, each K*N int4 codes +
    # K/G*N bf16 scales + K/G*N int4 zeros.
    def w4_matrix_bytes(self, K: int, N: int) -> int:
        return K * N // 2 + (K // self.group_size) * N * 2 + (K // self.group_size) * N // 2

    @property
    def expert_bytes(self) -> int:
        d, f = self.hidden, self.ffn
        return 2 * self.w4_matrix_bytes(d, f) + self.w4_matrix_bytes(f, d)

    @property
    def attn_bytes_per_layer(self) -> int:
        """W4 q|k|v and o projections (the paper's W4 model)."""
        d, hd = self.hidden, self.head_dim
        return (self.w4_matrix_bytes(d, (self.n_heads + 2 * self.n_kv_heads) * hd)
                + self.w4_matrix_bytes(self.n_heads * hd, d))

    @property
    def non_moe_bytes(self) -> int:
        d = self.hidden
        per_layer = self.attn_bytes_per_layer + self.num_experts * d * 2 + 2 * d * 2
        return self.num_layers * per_layer + 2 * self.vocab * d * 2 + d * 2

    @property
    def total_bytes(self) -> int:
        return self.non_moe_bytes + self.num_layers * self.num_experts * self.expert_bytes


def shape_names() -> list[str]:
    return sorted(p.stem for p in (_HERE / "shapes").glob("*.json"))


def load_shape(name: str) -> ModelShape:
    p = _HERE / "shapes" / f"{name}.json"
    if not p.is_file():
        raise ConfigError(f"unknown shape {name!r}; available: {shape_names()}")
    doc = json.loads(p.read_text(encoding="utf-8"))
    try:
        return ModelShape(**doc)
    except TypeError as e:
        raise ConfigError(f"{p}: {e}") from e


def model_config_for_shape(shape: ModelShape, predictor_mem_bytes: int = 0,
                           kv_reserve_bytes: int = 0) -> ModelConfig:
    """Reference-schema ModelConfig whose byte budget is the executed model's."""
    return ModelConfig(name=shape.name, num_layers=shape.num_layers, num_experts=shape.num_experts,
                       top_k=shape.top_k, total_param_bytes=shape.total_bytes,
                       non_moe_bytes=shape.non_moe_bytes, predictor_mem_bytes=predictor_mem_bytes,
                       kv_reserve_bytes=kv_reserve_bytes)

"""Co-located training apps for the configs of BASELINE.json.

* linear problems   -- the reference's own numeric workload (equivalence.py:42-147):
                       least squares / logistic regression, dim 8, seeded datasets.
* MLP 784-256-10    -- config 1 (cross-entropy, batch 64 per worker).
* ResNet-50, VGG-16, BERT-base -- configs 2/3/5 (bf16 autocast, fp32 master
                       parameters and gradients, synthetic data).

Host-side data generation uses the reference's seeding scheme verbatim in
meaning (equivalence.py:84-132): dataset ``default_rng(dataset_seed)``, initial
parameters ``default_rng([seed, 0])``, mini-batch indices
``default_rng([seed, 1, t, worker]).integers(0, size, batch)``.  That is
*input* generation only: all index arrays and datasets are uploaded once and
every gather, forward, backward and update runs on the device.
"""

from __future__ import annotations

import contextlib
import math
from dataclasses import dataclass
from typing import Sequence
from enum import Enum

import numpy as np
import torch
import torch.nn.functional as F

from .fusion import SgdSettings, flatten_parameters
from .scheduler import App


def _world() -> int:
    import torch.distributed as dist

    return dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1


def _flatten(params, flat):
    """flatten_parameters for the sharded / p2p sync (shards = world size); None when not asked.

    ``flat`` is False, True (torch allocation, sharded NCCL sync), "ipc" (cudaMalloc'd,
    mappable by peers, p2p / ce sync) or "nvls" (bound to an NVSwitch multicast object)."""
    if not flat:
        return None
    return flatten_parameters(params, 32, _world(), ipc="nvls" if flat == "nvls" else (flat == "ipc"))[0]

__all__ = [
    "LossKind",
    "SgdConfig",
    "make_dataset",
    "initial_parameters",
    "batch_indices",
    "LinearModel",
    "linear_app",
    "MlpConfig",
    "make_mlp_dataset",
    "mlp_initial_parameters",
    "mlp_app",
    "resnet50_app",
    "vgg16_app",
    "bert_app",
    "synthetic_image_batches",
    "synthetic_app",
    "fixed_time_app",
]


# ---------------------------------------------------------------------------
# the reference's linear problems
# ---------------------------------------------------------------------------
class LossKind(Enum):
    LEAST_SQUARES = "least_squares"
    LOGISTIC = "logistic_regression"


@dataclass(frozen=True)
class SgdConfig:
    """Synchronous-SGD setup of one linear job (equivalence.py:47-65)."""

    learning_rate: float
    workers: int
    loss: LossKind
    dataset_seed: int
    dim: int = 8
    dataset_size: int = 128
    batch_size: int = 16

    def __post_init__(self):
        if self.learning_rate <= 0:
            raise ValueError("learning_rate must be > 0")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if min(self.dim, self.dataset_size, self.batch_size) < 1:
            raise ValueError("dim, dataset_size and batch_size must be >= 1")


def make_dataset(config: SgdConfig) -> tuple[np.ndarray, np.ndarray]:
    """Seeded synthetic dataset (equivalence.py:84-95 seeding)."""
    rng = np.random.default_rng(config.dataset_seed)
    x = rng.standard_normal((config.dataset_size, config.dim))
    z = x @ rng.standard_normal(config.dim)
    y = z if config.loss is LossKind.LEAST_SQUARES else (z > 0).astype(np.float64)
    return x, y


def initial_parameters(dim: int, rng_seed: int) -> np.ndarray:
    """equivalence.py:98-100 seeding: default_rng([seed, 0]).standard_normal(dim)."""
    return np.random.default_rng([rng_seed, 0]).standard_normal(dim)


def batch_indices(rng_seed: int, iteration: int, worker: int, dataset_size: int,
                  batch_size: int) -> np.ndarray:
    """equivalence.py:129-132 seeding for the mini-batch of (iteration, worker)."""
    rng = np.random.default_rng([rng_seed, 1, iteration, worker])
    return rng.integers(0, dataset_size, size=batch_size)


def _index_table(rng_seed: int, iterations: int, workers: int, size: int, batch: int) -> np.ndarray:
    out = np.empty((iterations, workers, batch), dtype=np.int64)
    for t in range(iterations):
        for w in range(workers):
            out[t, w] = batch_indices(rng_seed, t + 1, w, size, batch)
    return out


class LinearModel(torch.nn.Module):
    def __init__(self, init: np.ndarray):
        super().__init__()
        self.weight = torch.nn.Parameter(torch.as_tensor(init, dtype=torch.float32).clone())


def _linear_loss(kind: LossKind):
    def loss_fn(model: LinearModel, batch):
        x, y = batch
        z = x @ model.weight
        if kind is LossKind.LEAST_SQUARES:
            r = z - y
            return 0.5 * torch.mean(r * r)
        return torch.mean(F.softplus(z) - y * z)   # logaddexp(0, z) - y z
    return loss_fn


class _GatherData:
    """data(t, worker) -> (x[idx], y[idx]) gathered on the device."""

    def __init__(self, x: torch.Tensor, y: torch.Tensor, idx: torch.Tensor):
        self.x, self.y, self.idx = x, y, idx

    def __call__(self, t: int, worker: int):
        sel = self.idx[t - 1, worker]
        return self.x.index_select(0, sel), self.y.index_select(0, sel)

    def graph(self, t_dev: torch.Tensor, worker: int):
        """The same batch with the iteration read from a device tensor (CUDA-graph replays)."""
        sel = self.idx[:, worker].index_select(0, t_dev - 1).view(-1)
        return self.x.index_select(0, sel), self.y.index_select(0, sel)


def linear_app(config: SgdConfig, job_id: str, rng_seed: int, iterations: int,
               device: torch.device, local_workers: int | None = None, momentum: float = 0.0,
               flat=False) -> App:
    """One of the reference's synthetic SGD jobs as a device app (momentum: torch-SGD rule)."""
    x, y = make_dataset(config)
    idx = _index_table(rng_seed, iterations, config.workers, config.dataset_size, config.batch_size)
    model = LinearModel(initial_parameters(config.dim, rng_seed)).to(device)
    flat_params = _flatten(list(model.parameters()), flat)
    data = _GatherData(torch.as_tensor(x, dtype=torch.float32, device=device),
                       torch.as_tensor(y, dtype=torch.float32, device=device),
                       torch.as_tensor(idx, device=device))
    return App(job_id, model, _linear_loss(config.loss), data,
               SgdSettings(config.learning_rate, momentum=momentum), iterations,
               local_workers=config.workers if local_workers is None else local_workers,
               samples_per_batch=config.batch_size, flat_params=flat_params, data_graph=data.graph)


# ---------------------------------------------------------------------------
# config 1: MLP 784-256-10
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class MlpConfig:
    learning_rate: float = 0.05
    workers: int = 2
    dataset_seed: int = 0
    in_dim: int = 784
    hidden: int = 256
    classes: int = 10
    dataset_size: int = 4096
    batch_size: int = 64
    momentum: float = 0.0


def make_mlp_dataset(config: MlpConfig) -> tuple[np.ndarray, np.ndarray]:
    rng = np.random.default_rng(config.dataset_seed)
    x = rng.standard_normal((config.dataset_size, config.in_dim))
    y = rng.integers(0, config.classes, size=config.dataset_size)
    return x, y


def mlp_initial_parameters(config: MlpConfig, rng_seed: int) -> list[np.ndarray]:
    """[W1 (h, in), b1 (h), W2 (c, h), b2 (c)], N(0,1)/sqrt(fan_in), drawn in that order."""
    rng = np.random.default_rng([rng_seed, 0])
    s1, s2 = 1.0 / math.sqrt(config.in_dim), 1.0 / math.sqrt(config.hidden)
    w1 = rng.standard_normal((config.hidden, config.in_dim)) * s1
    b1 = rng.standard_normal(config.hidden) * s1
    w2 = rng.standard_normal((config.classes, config.hidden)) * s2
    b2 = rng.standard_normal(config.classes) * s2
    return [w1, b1, w2, b2]


def _mlp_module(config: MlpConfig, init: list[np.ndarray]) -> torch.nn.Module:
    m = torch.nn.Sequential(torch.nn.Linear(config.in_dim, config.hidden), torch.nn.ReLU(),
                            torch.nn.Linear(config.hidden, config.classes))
    with torch.no_grad():
        for p, v in zip(m.parameters(), init):
            p.copy_(torch.as_tensor(v, dtype=torch.float32))
    return m


def _ce_loss(model, batch):
    x, y = batch
    return F.cross_entropy(model(x), y)


def mlp_app(config: MlpConfig, job_id: str, rng_seed: int, iterations: int,
            device: torch.device, local_workers: int | None = None,
            worker_count: int | None = None, flat: bool = False, graphed: bool = False) -> App:
    """Config 1 app: two of these co-located, W = 2, batch 64 per worker.  ``graphed``: forward and
    backward as CUDA graphs (fp32), so the gradients come back in static buffers (p2p_gather)."""
    x, y = make_mlp_dataset(config)
    workers = config.workers if worker_count is None else worker_count
    idx = _index_table(rng_seed, iterations, workers, config.dataset_size, config.batch_size)
    model = _mlp_module(config, mlp_initial_parameters(config, rng_seed)).to(device)
    flat_params = _flatten(list(model.parameters()), flat)   # before any graph captures the addresses
    if graphed:
        model = _GraphedImageModel(model, torch.zeros(config.batch_size, config.in_dim, device=device),
                                   autocast=False)
    data = _GatherData(torch.as_tensor(x, dtype=torch.float32, device=device),
                       torch.as_tensor(y, dtype=torch.int64, device=device),
                       torch.as_tensor(idx, device=device))
    return App(job_id, model, _ce_loss, data,
               SgdSettings(config.learning_rate, momentum=config.momentum), iterations,
               local_workers=config.workers if local_workers is None else local_workers,
               samples_per_batch=config.batch_size, flat_params=flat_params, data_graph=data.graph)


# ---------------------------------------------------------------------------
# configs 2/3/5: image / text models with synthetic data
# ---------------------------------------------------------------------------
class _CycleData:
    """Cycles through pre-built batches (device-resident or pinned host)."""

    def __init__(self, batches: list[tuple]):
        self.batches = batches
        self._stacked = None

    def __call__(self, t: int, worker: int):
        return self.batches[(t - 1) % len(self.batches)]

    def graph(self, t_dev: torch.Tensor, worker: int):
        """The same cycle with the iteration read from a device tensor (CUDA-graph replays): the
        batches are stacked once (4-D image tensors in their NHWC storage order, so the selected
        batch comes back as the same channels_last view) and indexed by (t - 1) mod n."""
        if self._stacked is None:
            def store(x):
                if x.dim() == 4 and x.is_contiguous(memory_format=torch.channels_last):
                    return x.permute(0, 2, 3, 1), True
                return x, False
            fields = list(zip(*self.batches))
            self._stacked = []
            for f in fields:
                parts = [store(x) for x in f]
                self._stacked.append((torch.stack([p for p, _ in parts]), parts[0][1]))
        n = len(self.batches)
        sel = torch.remainder(t_dev - 1, n)
        out = []
        for st, nhwc in self._stacked:
            x = st.index_select(0, sel)[0]
            out.append(x.permute(0, 3, 1, 2) if nhwc else x)
        return tuple(out)


def synthetic_image_batches(batch: int, n_batches: int, seed: int, device: torch.device,
                            host_uint8: bool = False, classes: int = 1000, size: int = 224):
    """Synthetic ImageNet-shaped batches.

    device mode: bf16 N(0,1) images [B,3,H,W] in channels_last + int64 labels on the GPU.
    host mode:   pinned uint8 NHWC images + labels (the e2e path copies them every step
                 and normalises on the device).
    """
    g = torch.Generator(device="cpu").manual_seed(seed)
    out = []
    for _ in range(n_batches):
        labels = torch.randint(0, classes, (batch,), generator=g)
        if host_uint8:
            img = torch.randint(0, 256, (batch, size, size, 3), dtype=torch.uint8, generator=g)
            out.append((img.pin_memory(), labels.pin_memory()))
        else:
            gd = torch.Generator(device=device).manual_seed(seed + len(out))
            img = torch.randn((batch, 3, size, size), generator=gd, device=device,
                              dtype=torch.bfloat16).contiguous(memory_format=torch.channels_last)
            out.append((img, labels.to(device)))
    return out


def _image_loss(model, batch):
    x, y = batch
    if x.dtype == torch.uint8:   # e2e path: NHWC bytes -> normalised bf16 channels_last
        x = x.permute(0, 3, 1, 2).to(torch.bfloat16).sub_(127.5).mul_(1.0 / 64.0)
    return F.cross_entropy(model(x), y)


class _GraphedImageModel(torch.nn.Module):
    """Forward and backward of a model captured as two CUDA graphs.

    torch.cuda.make_graphed_callables captures the forward and the backward
    separately, so the scheduler can still record the forward/backward span
    boundary between the two replays; parameters stay the module's own
    tensors (K2 updates them in place and the next replay reads the new
    values), inputs are copied into the graph's static input buffer, and the
    gradients come back in static graph memory -- stable addresses that the
    scheduler keeps alive until the app's K2 has consumed them.
    """

    def __init__(self, model: torch.nn.Module, sample: torch.Tensor, autocast: bool = True):
        super().__init__()
        self.inner = model
        quiet = getattr(torch.autograd.graph, "set_warn_on_accumulate_grad_stream_mismatch", None)
        if quiet is not None:  # capture runs on a side stream by design
            quiet(False)
        amp = (torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False) if autocast
               else contextlib.nullcontext())
        with amp:
            self.graphed = torch.cuda.make_graphed_callables(model, (sample,), num_warmup_iters=3)

    def forward(self, x):
        return self.graphed(x)


def _image_app(model: torch.nn.Module, job_id: str, batch: int, iterations: int,
               device: torch.device, seed: int, host_data: bool, sgd: SgdSettings,
               n_batches: int = 2, graphed: bool = False, flat: bool = False,
               fast_bn: bool = False, stem: str = "gemm") -> App:
    if fast_bn:   # NHWC BatchNorm kernels of libcrossover.so instead of ATen's (same semantics)
        from .bn import fuse_resnet, swap_batchnorm

        swap_batchnorm(model)
        if hasattr(model, "layer1"):
            fuse_resnet(model)      # BN + ReLU (+ residual add) in one pass
    if stem == "gemm":   # RGB stem as im2col + tensor-core GEMMs instead of cuDNN (stem.py)
        from .stem import gemm_stem

        gemm_stem(model)
    model = model.to(device).to(memory_format=torch.channels_last)
    data = _CycleData(synthetic_image_batches(batch, n_batches, seed, device, host_uint8=host_data))
    params = [p for p in model.parameters() if p.requires_grad]
    flat_params = _flatten(params, flat)          # before any graph captures the addresses
    if graphed:
        sample = torch.randn((batch, 3, 224, 224), device=device, dtype=torch.bfloat16
                             ).contiguous(memory_format=torch.channels_last)
        model = _GraphedImageModel(model, sample)
    return App(job_id, model, _image_loss, data, sgd, iterations, params=params,
               autocast_dtype=torch.bfloat16, samples_per_batch=batch,
               autocast_cache=not graphed, flat_params=flat_params,
               data_graph=None if host_data else data.graph)


DEFAULT_IMAGE_SGD = SgdSettings(lr=0.1, momentum=0.9, weight_decay=1e-4)
# VGG-16 has no BatchNorm: the torchvision recipe trains it at lr 0.01 / weight decay 5e-4; at
# lr 0.1 it diverges within ~13 steps on synthetic data (weights -> NaN), which invalidates any
# throughput measured afterwards (tools/diag_mix3.py)
VGG_SGD = SgdSettings(lr=0.01, momentum=0.9, weight_decay=5e-4)


def resnet50_app(job_id: str, batch: int, iterations: int, device: torch.device, seed: int = 0,
                 host_data: bool = False, sgd: SgdSettings = DEFAULT_IMAGE_SGD,
                 graphed: bool = False, flat: bool = False, fast_bn: bool = False,
                 stem: str = "gemm", data_seed: int | None = None) -> App:
    """``seed`` initialises the weights -- the same on every rank (data-parallel replicas);
    ``data_seed`` (default ``seed``) draws this worker's synthetic batches -- per rank."""
    import torchvision

    torch.manual_seed(seed)
    return _image_app(torchvision.models.resnet50(), job_id, batch, iterations, device,
                      seed if data_seed is None else data_seed, host_data, sgd, graphed=graphed,
                      flat=flat, fast_bn=fast_bn, stem=stem)


def vgg16_app(job_id: str, batch: int, iterations: int, device: torch.device, seed: int = 0,
                 host_data: bool = False, sgd: SgdSettings = VGG_SGD,
                 graphed: bool = False, flat: bool = False, fast_bn: bool = False,
                 stem: str = "gemm", data_seed: int | None = None) -> App:
    """Weights from ``seed`` (identical replicas), batches from ``data_seed`` (per rank)."""
    import torchvision

    torch.manual_seed(seed)
    return _image_app(torchvision.models.vgg16(), job_id, batch, iterations, device,
                      seed if data_seed is None else data_seed, host_data, sgd, graphed=graphed,
                      flat=flat, fast_bn=fast_bn, stem=stem)


def bert_app(job_id: str, batch: int, seq_len: int, iterations: int, device: torch.device,
             seed: int = 0, sgd: SgdSettings = SgdSettings(lr=1e-4, momentum=0.9),
             flat=False, data_seed: int | None = None) -> App:
    """BERT-base encoder (transformers BertModel defaults) with a masked-token-style loss.
    Weights from ``seed`` (identical replicas), token batches from ``data_seed`` (per rank)."""
    from transformers import BertConfig, BertModel

    torch.manual_seed(seed)
    cfg = BertConfig()
    model = BertModel(cfg, add_pooling_layer=True).to(device)
    head = torch.nn.Linear(cfg.hidden_size, cfg.vocab_size, bias=False).to(device)
    g = torch.Generator(device="cpu").manual_seed(seed if data_seed is None else data_seed)
    ids = torch.randint(0, cfg.vocab_size, (batch, seq_len), generator=g).to(device)
    labels = torch.randint(0, cfg.vocab_size, (batch, seq_len), generator=g).to(device)

    class _Wrap(torch.nn.Module):
        def __init__(self):
            super().__init__()
            self.bert, self.head = model, head

    wrap = _Wrap()
    flat_params = _flatten([p for p in wrap.parameters() if p.requires_grad], flat)

    def loss_fn(m, b):
        i, lab = b
        h = m.bert(input_ids=i).last_hidden_state
        return F.cross_entropy(m.head(h).float().view(-1, cfg.vocab_size), lab.view(-1))

    data = _CycleData([(ids, labels)])
    return App(job_id, wrap, loss_fn, data, sgd, iterations,
               autocast_dtype=torch.bfloat16, samples_per_batch=batch, flat_params=flat_params,
               data_graph=data.graph)


# ---------------------------------------------------------------------------
# config 4: synthetic bucket of S bytes vs a fixed compute kernel
# ---------------------------------------------------------------------------
class _SyntheticModel(torch.nn.Module):
    def __init__(self, numels: list[int], seed: int, device):
        super().__init__()
        g = torch.Generator(device="cpu").manual_seed(seed)
        self.weights = torch.nn.ParameterList(
            [torch.nn.Parameter((torch.randn(n, generator=g) * 0.01).to(device)) for n in numels])
        self.coef = [torch.randn(n, generator=g).to(device) for n in numels]


def synthetic_app(job_id: str, bucket_bytes: int, iterations: int, device: torch.device,
                  gemm_n: int = 8192, gemm_reps: int = 3, n_tensors: int = 16, seed: int = 0,
                  sgd: SgdSettings = SgdSettings(lr=1e-3), flat: bool = False,
                  tensor_bytes: Sequence[int] | None = None) -> App:
    """An app whose compute is a fixed bf16 GEMM chain (gemm_reps x [n,n]@[n,n]) and whose
    fused gradient is `bucket_bytes` of fp32 (mirrors cli._payload_for_ratio, cli.py:79-98:
    the sweep dials the payload against a fixed compute time).  ``tensor_bytes`` gives the
    exact per-tensor payload instead (a scenario job's split, scenario.py:114-119); each
    tensor holds ceil(bytes / 4) fp32 elements, at least one."""
    if tensor_bytes is not None:
        sizes = [max(1, (int(b) + 3) // 4) for b in tensor_bytes]
    else:
        numel = max(bucket_bytes // 4, n_tensors)
        sizes = [numel // n_tensors] * n_tensors
        sizes[-1] += numel - sum(sizes)
    model = _SyntheticModel(sizes, seed, device)
    g = torch.Generator(device=device).manual_seed(seed)
    a = torch.randn(gemm_n, gemm_n, device=device, dtype=torch.bfloat16, generator=g)
    b = torch.randn(gemm_n, gemm_n, device=device, dtype=torch.bfloat16, generator=g) / gemm_n ** 0.5

    def loss_fn(m, batch):
        x = a
        with torch.no_grad():
            for _ in range(gemm_reps):
                x = x @ b
        s = sum((w * c).sum() for w, c in zip(m.weights, m.coef))
        return s + x[0, 0].float() * 0.0

    flat_params = _flatten(list(model.weights), flat)
    return App(job_id, model, loss_fn, lambda t, w: (), sgd, iterations, samples_per_batch=1,
               flat_params=flat_params)


# ---------------------------------------------------------------------------
# apps of known compute duration (timing-level schedule tests, comm/comp sweeps)
# ---------------------------------------------------------------------------
class _FixedTimePhase(torch.autograd.Function):
    """Forward and backward that each take a fixed device time (cs_spin_ns) and hand back
    preallocated gradients: the app's compute is exactly `forward_ns + backward_ns` of device time
    on one SM, with no memory traffic, so measured schedules can be compared with the reference's
    recurrences in its own units (JobProfile.forward_time / backward_time, workload.py:43-56)."""

    @staticmethod
    def forward(ctx, forward_ns, backward_ns, grads, gemm, *weights):
        ctx.backward_ns, ctx.grads, ctx.gemm = backward_ns, grads, gemm
        _FixedTimePhase._compute(forward_ns, gemm, weights[0].device)
        return weights[0].new_zeros(())

    @staticmethod
    def backward(ctx, _dloss):
        _FixedTimePhase._compute(ctx.backward_ns, ctx.gemm, ctx.grads[0].device)
        return (None, None, None, None, *ctx.grads)

    @staticmethod
    def _compute(amount, gemm, device):
        """`amount` ns of spin on one SM, or (gemm = (a, b)) `amount` chained bf16 GEMMs."""
        if gemm is None:
            from . import _lib

            _lib.spin_ns(amount, torch.cuda.current_stream(device).cuda_stream)
            return
        a, b = gemm
        with torch.no_grad():
            x = a
            for _ in range(int(amount)):
                x = x @ b


class _FixedTimeModel(torch.nn.Module):
    def __init__(self, numels: list[int], device, seed: int):
        super().__init__()
        g = torch.Generator(device="cpu").manual_seed(seed)

        def tile(numel, scale):   # small seeded block on the host, tiled on the device
            base = min(numel, 1 << 20)
            reps = (numel + base - 1) // base
            return (torch.randn(base, generator=g) * scale).to(device).repeat(reps)[:numel].clone()

        self.weights = torch.nn.ParameterList([torch.nn.Parameter(tile(n, 0.01)) for n in numels])
        # the gradients K1 / K2 consume every iteration (fixed values, fixed addresses)
        self.grads = tuple(tile(n, 1e-3) for n in numels)


def fixed_time_app(job_id: str, forward_ns: int, backward_ns: int, bucket_bytes: int, iterations: int,
                   device: torch.device, seed: int = 0, sgd: SgdSettings = SgdSettings(lr=1e-3, momentum=0.9),
                   flat=False, samples_per_batch: int = 1,
                   tensor_bytes: Sequence[int] | None = None, gemm_n: int = 0) -> App:
    """An app whose forward / backward take `forward_ns` / `backward_ns` of device time and whose
    fused gradient is `bucket_bytes` of fp32 (one tensor, or the exact split ``tensor_bytes`` of a
    scenario job, scenario.py:114-119).  The sync is the real one (K1 / NVLink transport / K2 over
    the bucket), so its duration is dialed by the bucket size the way cli._payload_for_ratio
    (cli.py:79-98) dials the payload against a fixed compute time.

    ``gemm_n > 0`` replaces the spin kernel by real tensor-core work of fixed size: forward_ns /
    backward_ns are then COUNTS of chained bf16 [n, n] @ [n, n] GEMMs (the gradient stays the
    preallocated one, so the compute does not grow with the bucket)."""
    sizes = ([max(1, (int(b) + 3) // 4) for b in tensor_bytes] if tensor_bytes is not None
             else [max(1, int(bucket_bytes) // 4)])
    model = _FixedTimeModel(sizes, device, seed)
    params = list(model.weights)
    flat_params = _flatten(params, flat)
    fwd, bwd = int(forward_ns), int(backward_ns)
    gemm = None
    if gemm_n:
        g = torch.Generator(device=device).manual_seed(seed)
        gemm = (torch.randn(gemm_n, gemm_n, device=device, dtype=torch.bfloat16, generator=g),
                torch.randn(gemm_n, gemm_n, device=device, dtype=torch.bfloat16, generator=g) / gemm_n ** 0.5)

    def loss_fn(m, batch):
        return _FixedTimePhase.apply(fwd, bwd, m.grads, gemm, *m.weights)

    return App(job_id, model, loss_fn, lambda t, w: (), sgd, iterations,
               params=params, samples_per_batch=samples_per_batch, flat_params=flat_params,
               data_graph=lambda t_dev, w: ())

"""Workload / sweep definitions for BASELINE.json configs (input generation only).

Holds parameter *encodings* (integers handed to both sides), never the method's
arithmetic.  Cost constants are invented (the paper gives no latency model,
SPEC.md:133); see DESIGN.md "Invented cost constants" and SURVEY.md §8(c).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

from . import traces

# ---- enums shared by the binary contract (values fixed in include/continuum.h) ----
PRIO_PROG_FCFS, PRIO_REQ_FCFS, PRIO_PLAS = 0, 1, 2
PAUSE_EVICT, PAUSE_FIXED, PAUSE_PAPER, PAUSE_FITTED, PAUSE_INFERCEPT = 0, 1, 2, 3, 4
FLAG_VICTIMS_ANY = 1      # reading R13 alternative: victims whenever the head does not fit
FLAG_STEP_EXPIRY = 2      # reading R4 alternative: release pins only at scheduling points
ALWAYS = (1 << 63) - 1    # T_thresh sentinel: pin unconditionally (TTL grid policy)

STATUS_OK, STATUS_UNSCHEDULABLE, STATUS_EVENT_BUDGET = 0, 1, 2


def lq_from_delta(delta: float) -> int:
    """L_q = round(ln(3/delta) * 2^32): the Bernstein log factor in Q32 (SURVEY C-1)."""
    if not (0.0 < delta < 1.0):
        raise ValueError("delta must be in (0,1)")
    return int(round(math.log(3.0 / delta) * 2**32))


@dataclass(frozen=True)
class Engine:
    c0_ps: int
    c_pf_ps: int
    c_kv_ps: int
    c_h2d_ps: int
    bs: int = 16
    max_batch: int = 256
    dram_blocks: int = 0
    max_iters: int = (1 << 62)
    kv_growth: int = 0      # 0: reserve the request at admission (R12); 1: vLLM growth (R27-R30)
    prefill_chunk: int = 0  # 0: whole prompt in the first iteration; B: token budget (R31-R32)

    def as_array(self) -> np.ndarray:
        return np.array([self.c0_ps, self.c_pf_ps, self.c_kv_ps, self.c_h2d_ps, self.bs,
                         self.max_batch, self.dram_blocks, self.max_iters, self.kv_growth,
                         self.prefill_chunk], dtype=np.int64)


ENGINE_8B = Engine(c0_ps=2_000_000_000, c_pf_ps=13_400_000, c_kv_ps=16, c_h2d_ps=40_000_000)
ENGINE_70B_TP4 = Engine(c0_ps=5_000_000_000, c_pf_ps=29_400_000, c_kv_ps=10, c_h2d_ps=25_000_000,
                        dram_blocks=152_000)


@dataclass(frozen=True)
class Estimator:
    """Paper tunables + b + ttl_max."""
    delta: float = 0.05
    b_us: int = 60_000_000
    t_def_us: int = 10_000_000
    n_min: int = 5
    a_num: int = 1
    a_den: int = 10
    ttl_max_us: int = 50_000_000

    @property
    def lq(self) -> int:
        return lq_from_delta(self.delta)

    def as_array(self) -> np.ndarray:
        return np.array([self.lq, self.b_us, self.t_def_us, self.n_min, self.a_num, self.a_den,
                         self.ttl_max_us, 0], dtype=np.int64)


@dataclass(frozen=True)
class Policy:
    priority: int = PRIO_PROG_FCFS
    pause: int = PAUSE_EVICT
    dram: int = 0
    flags: int = 0
    t_pin_us: int = 0
    t_thresh_us: int = ALWAYS

    def as_array(self) -> np.ndarray:
        return np.array([self.priority, self.pause, self.dram, self.flags, self.t_pin_us,
                         self.t_thresh_us, 0, 0], dtype=np.int64)


# Named policies (SURVEY.md §8(a) policy matrix).
VLLM = Policy(PRIO_REQ_FCFS, PAUSE_EVICT)
VLLM_LMCACHE = Policy(PRIO_REQ_FCFS, PAUSE_EVICT, dram=1)
PROG_FCFS = Policy(PRIO_PROG_FCFS, PAUSE_EVICT)
CONTINUUM = Policy(PRIO_PROG_FCFS, PAUSE_PAPER)
CONTINUUM_FITTED = Policy(PRIO_PROG_FCFS, PAUSE_FITTED)
# comparison systems of the paper's evaluation (NEXT-1): Autellix PLAS and
# InferCept preserve/swap/evict on vLLM's request FCFS
AUTELLIX = Policy(PRIO_PLAS, PAUSE_EVICT)
INFERCEPT = Policy(PRIO_REQ_FCFS, PAUSE_INFERCEPT, dram=1)


def ttl_grid(tau_us: int) -> Policy:
    return Policy(PRIO_PROG_FCFS, PAUSE_FIXED, t_pin_us=int(tau_us), t_thresh_us=ALWAYS)


def simplified(t_pin_us: int, t_thresh_us: int) -> Policy:
    return Policy(PRIO_PROG_FCFS, PAUSE_FIXED, t_pin_us=int(t_pin_us), t_thresh_us=int(t_thresh_us))


@dataclass
class Sweep:
    """Mixed-radix sweep; replica r -> (seed, rate, kv, policy), policy fastest."""
    n_seeds: int
    gap_us: list[int]
    kv_blocks: list[int]
    policies: list[Policy]
    estimator: Estimator = field(default_factory=Estimator)
    fitted: np.ndarray | None = None   # int64 [F, J] TTL table for PAUSE_FITTED

    @property
    def n_replicas(self) -> int:
        return self.n_seeds * len(self.gap_us) * len(self.kv_blocks) * len(self.policies)

    @property
    def n_cells(self) -> int:
        return len(self.gap_us) * len(self.kv_blocks) * len(self.policies)

    def decode(self, r: int) -> tuple[int, int, int, int]:
        npol, nkv, nrate = len(self.policies), len(self.kv_blocks), len(self.gap_us)
        pol = r % npol
        kv = (r // npol) % nkv
        rate = (r // (npol * nkv)) % nrate
        seed = r // (npol * nkv * nrate)
        return seed, rate, kv, pol

    def policy_array(self) -> np.ndarray:
        return np.stack([p.as_array() for p in self.policies]).astype(np.int64)


@dataclass
class Workload:
    name: str
    trace: traces.TraceSet
    sweep: Sweep
    engine: Engine
    description: str = ""


def gap_from_jps(jps: float) -> int:
    return int(round(1e6 / jps))


def ttl_axis(n: int = 64, lo_us: int = 50_000, hi_us: int = 300_000_000) -> list[int]:
    """{0} ∪ (n-1) log-spaced TTLs in [lo, hi] (BASELINE config 3)."""
    v = np.rint(np.geomspace(lo_us, hi_us, n - 1)).astype(np.int64)
    return [0] + [int(x) for x in v]


def rate_axis(n: int = 64, lo: float = 0.02, hi: float = 2.0) -> list[int]:
    return [gap_from_jps(x) for x in np.geomspace(lo, hi, n)]


def config1() -> Workload:
    """1 replica set: 8 BFCL programs, 2k blocks, 8B, TTL vs evict (BASELINE configs[0])."""
    tr = traces.generate(1, 8, mix="bfcl", ctx_cap=2048 * 16)
    sw = Sweep(1, [gap_from_jps(0.5)], [2048], [CONTINUUM, PROG_FCFS, VLLM])
    return Workload("cfg1_bfcl8", tr, sw, ENGINE_8B, "8 BFCL programs, 2048 blocks, 8B costs")


def config2(n_seeds: int = 4096) -> Workload:
    """SWE-shaped, 200 programs, lambda=0.13 JPS, 16k blocks, PROG_FCFS+PAPER TTL (configs[1])."""
    tr = traces.generate(n_seeds, 200, mix="swe", ctx_cap=16384 * 16)
    sw = Sweep(n_seeds, [gap_from_jps(0.13)], [16384], [CONTINUUM])
    return Workload("cfg2_swe200x%d" % n_seeds, tr, sw, ENGINE_8B,
                    "200 SWE programs x %d seeds, 0.13 JPS, 16384 blocks, Continuum" % n_seeds)


def config3(n_seeds: int = 256, n_rates: int = 64, n_ttls: int = 64) -> Workload:
    """Arrival-rate x TTL-grid sweep on a 16 BFCL + 16 SWE mix, 8192 blocks (configs[2])."""
    tr = traces.generate(n_seeds, 32, n_bfcl=16, mix="mix", ctx_cap=8192 * 16)
    sw = Sweep(n_seeds, rate_axis(n_rates), [8192], [ttl_grid(t) for t in ttl_axis(n_ttls)])
    return Workload("cfg3_ttl_sweep_%dx%dx%d" % (n_rates, n_ttls, n_seeds), tr, sw, ENGINE_8B,
                    "%d rates x %d TTLs x %d seeds, 16 BFCL + 16 SWE, 8192 blocks" % (n_rates, n_ttls, n_seeds))


def config4(n_seeds: int = 4096) -> Workload:
    """70B TP=4 costs, DRAM tier, pools {97k, 24k}, 4 policies incl. FITTED (configs[3])."""
    tr = traces.generate(n_seeds, 32, n_bfcl=16, mix="mix", ctx_cap=24_000 * 16)
    pols = [VLLM_LMCACHE, replace(PROG_FCFS, dram=1), replace(CONTINUUM, dram=1),
            replace(CONTINUUM_FITTED, dram=1)]
    sw = Sweep(n_seeds, [gap_from_jps(0.13)], [97_000, 24_000], pols)
    return Workload("cfg4_70b_dram", tr, sw, ENGINE_70B_TP4, "70B TP4 costs + DRAM tier")


def config5(n_seeds: int = 256) -> Workload:
    """16 (policy x TTL) x 16 KV budgets x 16 rates x 256 seeds = 2^20 replicas (configs[4])."""
    tr = traces.generate(n_seeds, 32, n_bfcl=16, mix="mix", ctx_cap=1024 * 16)
    pols = [VLLM, PROG_FCFS, CONTINUUM, simplified(5_000_000, 2_000_000)]
    pols += [ttl_grid(t) for t in ttl_axis(13, 100_000, 60_000_000)[1:]]
    kv = [int(x) for x in np.rint(np.geomspace(1024, 65536, 16))]
    sw = Sweep(n_seeds, rate_axis(16), kv, pols)
    return Workload("cfg5_policy_sweep", tr, sw, ENGINE_8B, "16x16x16x%d policy sweep" % n_seeds)


# cfg4's FITTED policy replays the table ct_fit_ttl computes on the trace's own tool samples with
# these cost parameters (parameter encodings only; the fit itself is the library's / oracle's)
CFG4_FIT = {"J": 8, "ctx_j": [2000 * (j + 1) for j in range(8)], "w_j": [j + 1 for j in range(8)],
            "c_pin": 200, "a_num": 1, "a_den": 10, "step": 50_000, "K": 256}


def cfg4_fit_cost(engine: Engine) -> list[int]:
    """[c_pf, c_pin, bs, a_num, a_den, grid_step, K, J] for config 4's fit."""
    p = CFG4_FIT
    return [engine.c_pf_ps, p["c_pin"], engine.bs, p["a_num"], p["a_den"], p["step"], p["K"], p["J"]]


CONFIGS = {"1": config1, "2": config2, "3": config3, "4": config4, "5": config5}

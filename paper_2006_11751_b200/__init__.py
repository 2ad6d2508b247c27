"""B200-native APPO hot path (Sample Factory, arXiv 2006.11751).

Python host mirror of the reference's hot-path interface over the C ABI in
include/appo_capi.h (libappo_b200.so, hand-written sm_100a CUDA).  Function
names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/appo): ``vtrace`` (offpolicy.hpp:61),
``nstep_returns`` (:182), ``total_loss`` (:224), ``log_prob_and_entropy``
(policy.hpp:262), ``optimizer_step`` (policy.hpp:431), the policy-worker batch
inference (orchestrator.hpp:602-673) and the learner step
(orchestrator.hpp:760-868).  Errors raise ContractError / ConfigError /
NumericError like the reference's exception taxonomy (common.hpp:20-45).

Device buffers are torch CUDA tensors (torch is only the allocator/stream
plumbing here); every computation runs in libappo_b200.so.  There is no CPU
fallback: importing this package on a machine without the built library
raises, and calls without a CUDA device raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libappo_b200.so")


class AppoError(RuntimeError):
    pass


class ContractError(AppoError):
    """Broken precondition (common.hpp:23-26)."""


class ConfigError(AppoError):
    """Invalid configuration (common.hpp:30-33)."""


class NumericError(AppoError):
    """Non-finite value where a finite one is required (common.hpp:37-40)."""


class ResourceError(AppoError):
    """CUDA / allocation failure."""


_ERRS = {1: ContractError, 2: ConfigError, 3: NumericError, 4: ResourceError}


def _load():
    global LIB_PATH
    alt = os.environ.get("APPO_LIB")  # A/B diagnostics: another in-tree build of this library
    if alt:
        LIB_PATH = os.path.abspath(alt)
        return C.CDLL(LIB_PATH)
    from . import _build
    if _build.needs_build():  # missing or older than its sources: rebuild in-tree
        _build.build()
    return C.CDLL(LIB_PATH)


_L = _load()

_vp = C.c_void_p
_i = C.c_int
_i64 = C.c_int64
_u64 = C.c_uint64
_f = C.c_float


class ModelDesc(C.Structure):
    _fields_ = [("obs_c", C.c_int32), ("obs_h", C.c_int32), ("obs_w", C.c_int32),
                ("n_actions", C.c_int32), ("T", C.c_int32), ("reserved", C.c_int32 * 3)]

    @staticmethod
    def doom(n_actions: int = 6, T: int = 32) -> "ModelDesc":
        return ModelDesc(3, 72, 128, n_actions, T)

    @property
    def shape(self):
        return (self.obs_c, self.obs_h, self.obs_w, self.n_actions)

    @property
    def obs_dim(self):
        return self.obs_c * self.obs_h * self.obs_w


class HParams(C.Structure):
    _fields_ = [("lr", _f), ("beta1", _f), ("beta2", _f), ("eps", _f), ("grad_clip", _f),
                ("entropy_coef", _f), ("value_coef", _f), ("clip_low", _f), ("clip_high", _f),
                ("rho_bar", _f), ("c_bar", _f), ("gamma", _f), ("gae_lambda", _f),
                ("adv_source", C.c_int32), ("normalize_adv", C.c_int32),
                ("reserved", C.c_int32)]

    @staticmethod
    def defaults(**kw) -> "HParams":
        """Paper Table A.5 / reference defaults (policy.hpp:88-94, offpolicy.hpp:18-45,
        orchestrator.hpp:52-92)."""
        d = dict(lr=1e-4, beta1=0.9, beta2=0.999, eps=1e-6, grad_clip=4.0, entropy_coef=0.003,
                 value_coef=0.5, clip_low=1.0 / 1.1, clip_high=1.1, rho_bar=1.0, c_bar=1.0,
                 gamma=0.99, gae_lambda=0.95, adv_source=0, normalize_adv=0)
        d.update(kw)
        return HParams(**d)


def checkpoint_read(path: str, arrays: bool = True) -> dict:
    """Reads any APPOCKP1 file (also the reference's): header + f64 theta, m, v."""
    h, ver, t, n = _u64(), C.c_int64(), C.c_int64(), _u64(0)
    check(_L.appo_checkpoint_read_raw(os.fsencode(path), C.byref(h), C.byref(ver), C.byref(t),
                                      C.byref(n), None))
    out = {"spec_hash": h.value, "version": ver.value, "adam_t": t.value, "n": n.value}
    if arrays:
        buf = np.zeros(3 * n.value, dtype=np.float64)
        check(_L.appo_checkpoint_read_raw(os.fsencode(path), None, None, None, C.byref(n),
                                          buf.ctypes.data_as(C.c_void_p)))
        k = n.value
        out.update(theta=buf[:k], m=buf[k:2 * k], v=buf[2 * k:])
    return out


def model_spec_hash(desc) -> int:
    return int(_L.appo_model_spec_hash(C.byref(desc)))


def fnv1a64(data: bytes) -> int:
    b = bytes(data)
    return int(_L.appo_fnv1a64(C.c_char_p(b), len(b)))


class StepOut(C.Structure):
    _fields_ = [("policy_loss", C.c_double), ("value_loss", C.c_double),
                ("entropy", C.c_double), ("total_loss", C.c_double),
                ("mean_ratio", C.c_double), ("grad_norm", C.c_double),
                ("lag_mean", C.c_double), ("lag_max", C.c_double), ("version", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _sig(name, res, *args):
    f = getattr(_L, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("appo_last_error", C.c_char_p)
_sig("appo_checkpoint_save", _i, _vp, C.c_char_p)
_sig("appo_checkpoint_load", _i, _vp, C.c_char_p)
_sig("appo_checkpoint_read_raw", _i, C.c_char_p, C.POINTER(_u64), C.POINTER(C.c_int64),
     C.POINTER(C.c_int64), C.POINTER(_u64), _vp)
_sig("appo_model_spec_hash", _u64, C.POINTER(ModelDesc))
_sig("appo_fnv1a64", _u64, _vp, _u64)
_sig("appo_capi_version", _i)
_sig("appo_ctx_create", _i, C.POINTER(ModelDesc), _i, _u64, C.POINTER(_vp))
_sig("appo_ctx_destroy", _i, _vp)
_sig("appo_ctx_create_shared", _i, _vp, C.POINTER(_vp))
_sig("appo_ctx_set_sm_budget", _i, _vp, _i)
_sig("appo_ctx_set_pdl", _i, _vp, _i)
_sig("appo_ctx_set_learner_fork", _i, _vp, _i)
_sig("appo_ctx_set_stream", _i, _vp, _vp)
_sig("appo_ctx_sync", _i, _vp)
_sig("appo_ctx_launch_count", _i64, _vp)
_sig("appo_ctx_set_timing", _i, _vp, _i, C.c_char_p)
_sig("appo_ctx_timing_report", _i, _vp, C.c_char_p, _i)
_sig("appo_vtrace", _i, _vp, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _f, _f, _f, _vp, _vp, _vp,
     _vp)
_sig("appo_nstep_returns", _i, _vp, _i, _i, _vp, _vp, _vp, _f, _vp)
_sig("appo_gae", _i, _vp, _i, _i, _vp, _vp, _vp, _vp, _f, _f, _vp, _vp)
_sig("appo_total_loss", _i, _vp, _i, _vp, _vp, _vp, _vp, _vp, _f, _f, _f, _f,
     C.POINTER(C.c_double))
_sig("appo_logp_entropy", _i, _vp, _i, _i, _vp, _vp, _vp, _vp)
_sig("appo_sample_actions", _i, _vp, _i, _i, _vp, _u64, _u64, _vp, _vp)
_sig("appo_logp_entropy_heads", _i, _vp, _i, _i, _vp, _vp, _vp, _vp, _vp)
_sig("appo_sample_actions_heads", _i, _vp, _i, _i, _vp, _vp, _u64, _u64, _vp, _vp)
_sig("appo_adam_step", _i, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _f, _f, _f, _f, _f,
     C.POINTER(C.c_double))
_sig("appo_param_count", _i64, C.POINTER(ModelDesc))
_sig("appo_slot_layout", _i, C.POINTER(ModelDesc), C.POINTER(_u64))
_sig("appo_params_get", _i, _vp, _vp, C.POINTER(_i64))
_sig("appo_params_set", _i, _vp, _vp, _i64)
_sig("appo_adam_get", _i, _vp, _vp, _vp, C.POINTER(_i64))
_sig("appo_adam_set", _i, _vp, _vp, _vp, _i64)
_sig("appo_params_version", _i64, _vp)
_sig("appo_policy_forward", _i, _vp, _i, _vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp,
     C.POINTER(_i64))
_sig("appo_learner_step", _i, _vp, _vp, _u64, _vp, _i, C.POINTER(HParams), C.POINTER(StepOut))
_sig("appo_dbg_gemm", _i, _vp, _i, _i, _i, _vp, _i64, _i, _vp, _i64, _i, _vp, _i64, _i, _f, _vp,
     _vp, _i64, _i, _i)
_sig("appo_dbg_model_ptrs", _i, _vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp))
_sig("appo_dbg_copy_d2h", _i, _vp, _vp, _vp, _u64)
_sig("appo_dbg_ppo_loss", _i, _vp, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _f, _f, _f, _f, _vp,
     _vp)
_sig("appo_dbg_traj_loss", _i, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _f,
     _f, _f, _i, _f, _f, _f, _f, _f, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp)
_sig("appo_learner_submit", _i, _vp, _vp, _u64, _vp, _i, C.POINTER(HParams))
_sig("appo_learner_collect", _i, _vp, C.POINTER(StepOut))
_sig("appo_dp_unique_id", _i, C.c_char_p)
_sig("appo_dp_init", _i, _vp, _i, _i, C.c_char_p)
_sig("appo_dp_bucket_plan", _i, C.POINTER(ModelDesc), _vp, _i, C.POINTER(_i))
_sig("appo_sampler_create", _i, _vp, _i, _i, _u64, C.POINTER(_vp))
_sig("appo_sampler_destroy", _i, _vp)
_sig("appo_sampler_step", _i, _vp, _vp, _u64, C.c_int32, _i, _vp, _vp)
_sig("appo_sampler_set_ready_queue", _i, _vp, _vp)
_sig("appo_rollout_act", _i, _vp, _vp, _u64, C.c_int32, _i, _vp, _vp)
_sig("appo_rollout_wait", _i, _vp)
_sig("appo_rollout_feedback", _i, _vp, _vp, _u64, C.c_int32, _i, _vp, _vp, _vp)
_sig("appo_slotq_create", _i, _i, C.c_int32, C.c_int32, C.c_double, C.POINTER(_vp))
_sig("appo_slotq_destroy", _i, _vp)
_sig("appo_slotq_push", _i, _vp, _vp, _vp, _i)
_sig("appo_slotq_push_range", _i, _vp, _vp, C.c_int32, _i)
_sig("appo_slotq_pop", _i, _vp, _vp, _vp, _i)
_sig("appo_slotq_stats", _i, _vp, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64))
_sig("appo_params_copy", _i, _vp, _vp)
_sig("appo_params_export", _i, _vp, _vp)
_sig("appo_params_import", _i, _vp, _vp)
_sig("appo_pbt_create", _i, C.c_void_p, _i, _u64, _vp, C.POINTER(_vp))
_sig("appo_pbt_destroy", _i, _vp)
_sig("appo_pbt_controller_seed", _u64, _u64)
_sig("appo_pbt_record", _i, _vp, C.c_uint32, C.c_double)
_sig("appo_pbt_score", _i, _vp, C.c_uint32, C.POINTER(C.c_double), C.POINTER(_i))
_sig("appo_pbt_step", _i, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _i, C.POINTER(_i))
_sig("appo_pbt_tick", _i, _vp, _i64, _vp, _vp, _vp, _i, C.POINTER(_i), C.POINTER(_i))
_sig("appo_pbt_get_agent", _i, _vp, _i, _vp)
_sig("appo_pbt_max_events", _i, _vp)
_sig("appo_pbt_format_events", _i, _vp, _i, _i, C.c_char_p, _u64, C.POINTER(_u64))
_sig("appo_learner_submit_queued", _i, _vp, _vp, _u64, _vp, _vp, _i, C.POINTER(HParams))

LIB = _L


def check(status: int):
    if status != 0:
        msg = (_L.appo_last_error() or b"").decode(errors="replace")
        raise _ERRS.get(status, AppoError)(msg)


def param_count(desc: ModelDesc) -> int:
    return int(_L.appo_param_count(C.byref(desc)))


def slot_layout(desc: ModelDesc) -> dict:
    out = (_u64 * 10)()
    check(_L.appo_slot_layout(C.byref(desc), out))
    keys = ["obs", "hidden", "actions", "rewards", "logp", "dones", "versions", "boot_obs",
            "boot_hidden", "total"]
    return dict(zip(keys, [int(x) for x in out]))


def _ptr(t):
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ContractError("device tensors required (torch CUDA tensors)")


class Context:
    """One appo_ctx: a device, a stream, optional model (parameters + Adam)."""

    def __init__(self, device: int = 0, seed: int = 1, model: ModelDesc | None = None,
                 stream=None):
        import torch
        if not torch.cuda.is_available():
            raise ResourceError("libappo_b200 needs a CUDA device")
        self.torch = torch
        self.device = device
        self.model = model
        h = C.c_void_p()
        check(_L.appo_ctx_create(C.byref(model) if model is not None else None, device, seed,
                                 C.byref(h)))
        self.h = h
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        check(_L.appo_ctx_set_stream(self.h, C.c_void_p(self.stream.cuda_stream)))

    def shared(self, stream=None) -> "Context":
        """A context sharing this one's model on its own CUDA stream
        (appo_ctx_create_shared): run the sampler there concurrently with the
        learner on this context."""
        torch = self.torch
        c = Context.__new__(Context)
        c.torch = torch
        c.device = self.device
        c.model = self.model
        c._base = self  # keep the owner alive
        h = C.c_void_p()
        check(_L.appo_ctx_create_shared(self.h, C.byref(h)))
        c.h = h
        c.stream = stream if stream is not None else torch.cuda.Stream(self.device)
        check(_L.appo_ctx_set_stream(c.h, C.c_void_p(c.stream.cuda_stream)))
        return c

    def set_sm_budget(self, n_sms: int):
        check(_L.appo_ctx_set_sm_budget(self.h, n_sms))

    def set_pdl(self, enable: bool):
        """Programmatic dependent launch of this context's kernels."""
        check(_L.appo_ctx_set_pdl(self.h, int(enable)))

    def set_learner_fork(self, enable: bool):
        """Learner backward on two streams (weight gradients on a side stream)."""
        check(_L.appo_ctx_set_learner_fork(self.h, int(enable)))

    def close(self):
        if getattr(self, "h", None):
            _L.appo_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        check(_L.appo_ctx_sync(self.h))

    @property
    def launches(self) -> int:
        return int(_L.appo_ctx_launch_count(self.h))

    def set_timing(self, enable: bool, name_filter: str | None = None):
        check(_L.appo_ctx_set_timing(self.h, int(enable),
                                     name_filter.encode() if name_filter else None))

    def timing_report(self) -> list:
        """Per-kernel aggregated CUDA-event timing since set_timing (resets)."""
        import json
        buf = C.create_string_buffer(1 << 20)
        check(_L.appo_ctx_timing_report(self.h, buf, len(buf)))
        return [json.loads(l) for l in buf.value.decode().splitlines() if l.strip()]

    # ---- off-policy -----------------------------------------------------
    def vtrace(self, rewards, values, bootstrap, target_logp, behavior_logp, dones, gamma=0.99,
               rho_bar=1.0, c_bar=1.0, with_weights=False, sync=True):
        """vtrace (offpolicy.hpp:61-100) over [n_traj, T] tensors."""
        torch = self.torch
        _need_cuda(rewards, values, bootstrap, target_logp, behavior_logp, dones)
        n, T = rewards.shape
        v = torch.empty_like(rewards)
        pg = torch.empty_like(rewards)
        rho = torch.empty_like(rewards) if with_weights else None
        c = torch.empty_like(rewards) if with_weights else None
        check(_L.appo_vtrace(self.h, n, T, _ptr(rewards), _ptr(values), _ptr(bootstrap),
                             _ptr(target_logp), _ptr(behavior_logp), _ptr(dones), gamma, rho_bar,
                             c_bar, _ptr(v), _ptr(pg), _ptr(rho), _ptr(c)))
        if sync:
            self.sync()
        return (v, pg, rho, c) if with_weights else (v, pg)

    def nstep_returns(self, rewards, bootstrap, dones, gamma, sync=True):
        _need_cuda(rewards, bootstrap, dones)
        n, T = rewards.shape
        ret = self.torch.empty_like(rewards)
        check(_L.appo_nstep_returns(self.h, n, T, _ptr(rewards), _ptr(bootstrap), _ptr(dones),
                                    gamma, _ptr(ret)))
        if sync:
            self.sync()
        return ret

    def gae(self, rewards, values, bootstrap, dones, gamma, lam, sync=True):
        _need_cuda(rewards, values, bootstrap, dones)
        n, T = rewards.shape
        adv = self.torch.empty_like(rewards)
        ret = self.torch.empty_like(rewards)
        check(_L.appo_gae(self.h, n, T, _ptr(rewards), _ptr(values), _ptr(bootstrap),
                          _ptr(dones), gamma, lam, _ptr(adv), _ptr(ret)))
        if sync:
            self.sync()
        return adv, ret

    def total_loss(self, ratios, adv, values, v_targets, entropies, clip_low=1 / 1.1,
                   clip_high=1.1, value_coef=0.5, entropy_coef=0.003):
        """total_loss (offpolicy.hpp:146-168) -> dict(policy, value, entropy, total)."""
        _need_cuda(ratios, adv, values, v_targets, entropies)
        out = (C.c_double * 4)()
        check(_L.appo_total_loss(self.h, ratios.numel(), _ptr(ratios), _ptr(adv), _ptr(values),
                                 _ptr(v_targets), _ptr(entropies), clip_low, clip_high,
                                 value_coef, entropy_coef, out))
        return dict(policy=out[0], value=out[1], entropy=out[2], total=out[3])

    def log_prob_and_entropy(self, logits, actions, sync=True):
        _need_cuda(logits, actions)
        B, A = logits.shape
        lp = self.torch.empty(B, device=logits.device, dtype=self.torch.float32)
        en = self.torch.empty_like(lp)
        check(_L.appo_logp_entropy(self.h, B, A, _ptr(logits), _ptr(actions), _ptr(lp), _ptr(en)))
        if sync:
            self.sync()
        return lp, en

    def log_prob_and_entropy_heads(self, sizes, logits, actions, sync=True):
        """log_prob_and_entropy (policy.hpp:262-281) over factored heads
        ``sizes``: logits [B][sum(sizes)], actions int32 [B][n_heads]."""
        _need_cuda(logits, actions)
        sz = (C.c_int32 * len(sizes))(*sizes)
        B = logits.shape[0]
        lp = self.torch.empty(B, device=logits.device, dtype=self.torch.float32)
        en = self.torch.empty_like(lp)
        check(_L.appo_logp_entropy_heads(self.h, B, len(sizes), sz, _ptr(logits), _ptr(actions),
                                         _ptr(lp), _ptr(en)))
        if sync:
            self.sync()
        return lp, en

    def sample_actions_heads(self, sizes, logits, key, counter0=0, sync=True):
        """sample_action (policy.hpp:232-258) over factored heads: actions
        [B][n_heads], joint log-prob [B]; u(b, j) = U(key, counter0 + b*n + j)."""
        _need_cuda(logits)
        sz = (C.c_int32 * len(sizes))(*sizes)
        B = logits.shape[0]
        a = self.torch.empty((B, len(sizes)), device=logits.device, dtype=self.torch.int32)
        lp = self.torch.empty(B, device=logits.device, dtype=self.torch.float32)
        check(_L.appo_sample_actions_heads(self.h, B, len(sizes), sz, _ptr(logits), key, counter0,
                                           _ptr(a), _ptr(lp)))
        if sync:
            self.sync()
        return a, lp

    def sample_actions(self, logits, key, counter0=0, sync=True):
        _need_cuda(logits)
        B, A = logits.shape
        a = self.torch.empty(B, device=logits.device, dtype=self.torch.int32)
        lp = self.torch.empty(B, device=logits.device, dtype=self.torch.float32)
        check(_L.appo_sample_actions(self.h, B, A, _ptr(logits), key, counter0, _ptr(a), _ptr(lp)))
        if sync:
            self.sync()
        return a, lp

    def optimizer_step(self, theta, m, v, grad, t, lr=1e-4, beta1=0.9, beta2=0.999, eps=1e-6,
                       grad_clip=4.0):
        """optimizer_step (policy.hpp:431-455) on flat fp32 tensors; t is the
        step number after the increment.  Returns the pre-clip gradient norm."""
        _need_cuda(theta, m, v, grad)
        norm = C.c_double()
        check(_L.appo_adam_step(self.h, theta.numel(), _ptr(theta), _ptr(m), _ptr(v), _ptr(grad),
                                t, lr, beta1, beta2, eps, grad_clip, C.byref(norm)))
        return norm.value

    # ---- model ------------------------------------------------------------
    @property
    def n_params(self) -> int:
        return param_count(self.model)

    def get_params(self):
        th = np.zeros(self.n_params, dtype=np.float32)
        ver = C.c_int64()
        check(_L.appo_params_get(self.h, th.ctypes.data_as(C.c_void_p), C.byref(ver)))
        return th, ver.value

    def set_params(self, theta: np.ndarray, version: int = 0):
        th = np.ascontiguousarray(theta, dtype=np.float32)
        assert th.size == self.n_params
        check(_L.appo_params_set(self.h, th.ctypes.data_as(C.c_void_p), version))

    def get_adam(self):
        m = np.zeros(self.n_params, dtype=np.float32)
        v = np.zeros(self.n_params, dtype=np.float32)
        t = C.c_int64()
        check(_L.appo_adam_get(self.h, m.ctypes.data_as(C.c_void_p),
                               v.ctypes.data_as(C.c_void_p), C.byref(t)))
        return m, v, t.value

    def set_adam(self, m, v, t):
        m = np.ascontiguousarray(m, dtype=np.float32)
        v = np.ascontiguousarray(v, dtype=np.float32)
        check(_L.appo_adam_set(self.h, m.ctypes.data_as(C.c_void_p), v.ctypes.data_as(C.c_void_p),
                               t))

    @property
    def version(self) -> int:
        return int(_L.appo_params_version(self.h))

    def save_checkpoint(self, path: str):
        """save_checkpoint (policy.hpp:545-564), APPOCKP1 format."""
        check(_L.appo_checkpoint_save(self.h, os.fsencode(path)))

    def load_checkpoint(self, path: str):
        """load_checkpoint (policy.hpp:567-605): ConfigError on a shape mismatch."""
        check(_L.appo_checkpoint_load(self.h, os.fsencode(path)))

    def policy_forward(self, obs, h_in, rng_counter0=0, want_logits=False, out=None):
        """Batched inference: obs u8 [B, C*H*W], h_in f32 [B, 512] (CUDA) ->
        dict(actions, logp, h_out, values[, logits], version)."""
        torch = self.torch
        _need_cuda(obs, h_in)
        B = obs.shape[0]
        dev = obs.device
        if out is None:
            out = dict(actions=torch.empty(B, dtype=torch.int32, device=dev),
                       logp=torch.empty(B, dtype=torch.float32, device=dev),
                       h_out=torch.empty(B, 512, dtype=torch.float32, device=dev),
                       values=torch.empty(B, dtype=torch.float32, device=dev))
            if want_logits:
                out["logits"] = torch.empty(B, self.model.n_actions, dtype=torch.float32,
                                            device=dev)
        ver = C.c_int64()
        check(_L.appo_policy_forward(self.h, B, _ptr(obs), _ptr(h_in), rng_counter0,
                                     _ptr(out["actions"]), _ptr(out["logp"]), _ptr(out["h_out"]),
                                     _ptr(out["values"]), _ptr(out.get("logits")),
                                     C.byref(ver)))
        out["version"] = ver.value
        return out

    def learner_step(self, region, slot_bytes: int, slot_ids, hp: HParams | None = None):
        """One APPO learner step over trajectory slots (layout v2) in FIFO order."""
        _need_cuda(region)
        ids = np.ascontiguousarray(slot_ids, dtype=np.int32)
        hp = hp or HParams.defaults()
        out = StepOut()
        check(_L.appo_learner_step(self.h, _ptr(region), slot_bytes,
                                   ids.ctypes.data_as(C.c_void_p), ids.size, C.byref(hp),
                                   C.byref(out)))
        return out.as_dict()

    def learner_submit(self, region, slot_bytes: int, slot_ids, hp: HParams | None = None):
        """Enqueue one learner step without waiting (appo_learner_submit)."""
        ids = np.ascontiguousarray(slot_ids, dtype=np.int32)
        hp = hp or HParams.defaults()
        check(_L.appo_learner_submit(self.h, _ptr(region), slot_bytes,
                                     ids.ctypes.data_as(C.c_void_p), ids.size, C.byref(hp)))

    def learner_submit_queued(self, region, slot_bytes: int, ready_q: "SlotQueue",
                              free_q: "SlotQueue | None", n_traj: int,
                              hp: HParams | None = None):
        """Enqueue one learner step over the next n_traj slots of ``ready_q``
        (popped on the device, FIFO); the slots go to ``free_q`` afterwards."""
        _need_cuda(region)
        hp = hp or HParams.defaults()
        check(_L.appo_learner_submit_queued(self.h, _ptr(region), slot_bytes, ready_q.h,
                                            free_q.h if free_q is not None else None, n_traj,
                                            C.byref(hp)))

    def learner_collect(self):
        """Wait for submitted steps; stats of the last one (appo_learner_collect)."""
        out = StepOut()
        check(_L.appo_learner_collect(self.h, C.byref(out)))
        return out.as_dict()

    def model_ptrs(self):
        th, g, pb = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(_L.appo_dbg_model_ptrs(self.h, C.byref(th), C.byref(g), C.byref(pb)))
        return th.value, g.value, pb.value

    def grad(self) -> np.ndarray:
        """The last learner step's flat fp32 gradient (pre-clip), for tests."""
        _, g, _ = self.model_ptrs()
        out = np.zeros(self.n_params, dtype=np.float32)
        check(_L.appo_dbg_copy_d2h(self.h, out.ctypes.data_as(C.c_void_p), C.c_void_p(g),
                                   out.nbytes))
        return out

    def export_params(self) -> bytes:
        """appo_params_export: this learner's state as a handle for another process."""
        buf = C.create_string_buffer(STATE_HANDLE_BYTES)
        check(_L.appo_params_export(self.h, buf))
        return buf.raw

    def import_params(self, handle: bytes):
        """appo_params_import: take another process's exported learner state."""
        check(_L.appo_params_import(self.h, C.create_string_buffer(bytes(handle),
                                                                   STATE_HANDLE_BYTES)))

    def ppo_loss_injected(self, logits, values, actions, blogp, adv, vt, clip_low=1 / 1.1,
                          clip_high=1.1, value_coef=0.5, entropy_coef=0.003):
        """The learner's fused loss kernel on injected inputs (include/appo_internal.h):
        returns dlog [B][A+1] (dL/dlogits, dL/dV) and the 8 loss statistics."""
        _need_cuda(logits, values, actions, blogp, adv, vt)
        B, A = logits.shape
        import torch
        dlog = torch.empty(B, A + 1, dtype=torch.float32, device=logits.device)
        stats = np.zeros(8)
        check(_L.appo_dbg_ppo_loss(self.h, B, A, _ptr(logits), _ptr(values), _ptr(actions),
                                   _ptr(blogp), _ptr(adv), _ptr(vt), clip_low, clip_high,
                                   value_coef, entropy_coef, _ptr(dlog),
                                   stats.ctypes.data_as(C.c_void_p)))
        return dlog, stats

    def traj_loss_injected(self, T, core, wpi, bpi, wv, bv, actions, rewards, blogp, dones,
                           gamma=0.99, rho_bar=1.0, c_bar=1.0, adv_source=0, gae_lambda=0.95,
                           clip_low=1 / 1.1, clip_high=1.1, value_coef=0.5, entropy_coef=0.003):
        """The learner's fused per-trajectory loss block (traj_loss_kernel) on injected
        core rows [B + n_traj][512] and head weights (include/appo_internal.h)."""
        _need_cuda(core, wpi, bpi, wv, bv, actions, rewards, blogp, dones)
        import torch
        R = core.shape[0]
        n = R // (T + 1)
        B = n * T
        A = wpi.shape[0]
        f = lambda *shape: torch.empty(*shape, dtype=torch.float32, device=core.device)
        out = dict(logits=f(R, A), values=f(R), vt=f(B), pg=f(B), adv=f(B), dcore=f(B, 512),
                   ghead=f(A * 512 + A + 512 + 1))
        stats = np.zeros(8)
        check(_L.appo_dbg_traj_loss(self.h, n, T, A, _ptr(core), _ptr(wpi), _ptr(bpi), _ptr(wv),
                                    _ptr(bv), _ptr(actions), _ptr(rewards), _ptr(blogp),
                                    _ptr(dones), gamma, rho_bar, c_bar, adv_source, gae_lambda,
                                    clip_low, clip_high, value_coef, entropy_coef,
                                    _ptr(out["logits"]), _ptr(out["values"]), _ptr(out["vt"]),
                                    _ptr(out["pg"]), _ptr(out["adv"]), _ptr(out["dcore"]),
                                    _ptr(out["ghead"]), stats.ctypes.data_as(C.c_void_p)))
        out["stats"] = stats
        return out

    def gemm(self, M, N, K, a, lda, a_mn, b, ldb, b_mn, out, ldo, flags=0, scale=1.0, bias=None,
             aux=None, ld_aux=0, bn=128, splits=1):
        """Engine-level GEMM hook (include/appo_internal.h) for tests."""
        check(_L.appo_dbg_gemm(self.h, M, N, K, _ptr(a), lda, int(a_mn), _ptr(b), ldb, int(b_mn),
                               _ptr(out), ldo, flags, scale, _ptr(bias), _ptr(aux), ld_aux, bn,
                               splits))


def dp_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(_L.appo_dp_unique_id(buf))
    return buf.raw


def dp_init(ctx: Context, dist, rank: int, world: int):
    """Join ``ctx`` to a data-parallel learner group of ``world`` ranks: rank 0's
    NCCL id is broadcast over ``dist`` (torch.distributed), then every
    learner step all-reduces (averages) the gradient before clip + Adam."""
    obj = [dp_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    check(_L.appo_dp_init(ctx.h, world, rank, C.create_string_buffer(obj[0], 128)))


STATE_HANDLE_BYTES = 512


def pbt_exchange(ctx: "Context", dist, rank: int, dst: int, src: int):
    """copy_weights(dst, src) across processes (one policy learner per rank):
    called on EVERY rank with the same pair (each rank runs an identical PBT
    controller on all-gathered scores).  The source exports, the destination
    imports, and the barrier keeps the source from training until the copy
    is done (the pbt_lock pair of runner.hpp:217-218)."""
    if dst == src:
        return
    obj = [ctx.export_params() if rank == src else None]
    dist.broadcast_object_list(obj, src=src)
    if rank == dst:
        ctx.import_params(obj[0])
    dist.barrier()


def dp_bucket_plan(desc: ModelDesc) -> list:
    """The data-parallel gradient buckets in reduction order: [(offset, count)]."""
    buf = (C.c_int64 * 16)()
    n = C.c_int()
    check(_L.appo_dp_bucket_plan(C.byref(desc), C.cast(buf, C.c_void_p), 8, C.byref(n)))
    return [(buf[2 * i], buf[2 * i + 1]) for i in range(n.value)]


class Sampler:
    """Device synthetic envs + rollout writer (appo_sampler_*, include/appo_capi.h):
    ``step(store, slot_base, t)`` advances all envs one step, writing step t of
    env e's rollout into slot slot_base + e."""

    def __init__(self, ctx: Context, n_envs: int, episode_len: int = 256, seed: int = 1):
        self.ctx = ctx
        self.n_envs = n_envs
        h = C.c_void_p()
        check(_L.appo_sampler_create(ctx.h, n_envs, episode_len, seed, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            _L.appo_sampler_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, store, slot_base: int, t: int, h_obs=None, h_actions=None):
        """h_obs / h_actions: optional pinned host tensors (CPU-actor path)."""
        check(_L.appo_sampler_step(self.h, _ptr(store.region), store.slot_bytes, slot_base, t,
                                   _ptr(h_obs), _ptr(h_actions)))

    # ---- CPU actors: RolloutWorker::submit_group / step_group (two phases) ----
    def act(self, store, slot_base: int, t: int, h_obs, h_actions=None):
        """Step t's observations (host tensor [n_envs][obs_dim], pinned for an
        asynchronous copy) -> slot row t + batched inference; sampled actions
        into ``h_actions`` (host int32 [n_envs]), valid after ``wait()``."""
        if h_obs is None or h_obs.is_cuda:
            raise ContractError("rollout act: host observations required")
        check(_L.appo_rollout_act(self.h, _ptr(store.region), store.slot_bytes, slot_base, t,
                                  _ptr(h_obs), _ptr(h_actions)))

    def wait(self):
        """Blocks until the last act's actions are on the host and the caller's
        observation buffers are no longer read."""
        check(_L.appo_rollout_wait(self.h))

    def feedback(self, store, slot_base: int, t: int, h_rewards, h_dones, h_next_obs=None):
        """The env transition of step t: rewards (f32) and dones (u8) [n_envs]
        from host memory; at t == T-1 also the next observations (bootstrap)."""
        for x in (h_rewards, h_dones, h_next_obs):
            if x is not None and x.is_cuda:
                raise ContractError("rollout feedback: host tensors required")
        check(_L.appo_rollout_feedback(self.h, _ptr(store.region), store.slot_bytes, slot_base, t,
                                       _ptr(h_rewards), _ptr(h_dones), _ptr(h_next_obs)))

    def set_ready_queue(self, q: "SlotQueue | None"):
        """After step T-1 of a rollout the written slots are pushed to ``q``."""
        self._ready_q = q  # keep the queue alive while attached
        check(_L.appo_sampler_set_ready_queue(self.h, q.h if q is not None else None))


class SlotQueue:
    """Device FIFO of slot ids (appo_slotq_*): the ready queue between rollout
    writers and the learner (trajstore.hpp:293-331) or the free list."""

    def __init__(self, device: int, n_slots: int, capacity: int = 0, timeout_s: float = 2.0):
        h = C.c_void_p()
        check(_L.appo_slotq_create(device, n_slots, capacity, timeout_s, C.byref(h)))
        self.h = h
        self.n_slots = n_slots

    def close(self):
        if getattr(self, "h", None):
            _L.appo_slotq_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def push(self, ctx: Context, ids):
        """ids: int32 CUDA tensor, enqueued in order on ctx's stream."""
        _need_cuda(ids)
        check(_L.appo_slotq_push(ctx.h, self.h, _ptr(ids), ids.numel()))

    def push_range(self, ctx: Context, first: int, n: int):
        check(_L.appo_slotq_push_range(ctx.h, self.h, first, n))

    def pop(self, ctx: Context, n: int, out=None):
        import torch
        if out is None:
            out = torch.empty(n, dtype=torch.int32, device=f"cuda:{ctx.device}")
        check(_L.appo_slotq_pop(ctx.h, self.h, _ptr(out), n))
        return out

    def stats(self) -> dict:
        p, q, t = _i64(), _i64(), _i64()
        check(_L.appo_slotq_stats(self.h, C.byref(p), C.byref(q), C.byref(t)))
        return {"pushed": p.value, "popped": q.value, "timeouts": t.value,
                "size": p.value - q.value}


# ---------------------------------------------------------------- PBT
PBT_MAX_REWARD_WEIGHTS = 8
PBT_EVENTS = ("mutate", "exchange", "skip-threshold")


class PbtConfig(C.Structure):
    """PopulationConfig (population.hpp:22-37) + ScoreWindow capacity."""
    _fields_ = [("pbt_period", C.c_int64), ("mutate_fraction", C.c_double),
                ("mutation_rate", C.c_double), ("mutation_factor", C.c_double),
                ("replace_fraction", C.c_double), ("exchange_threshold", C.c_double),
                ("has_exchange_threshold", C.c_int32), ("window", C.c_int32)]

    @staticmethod
    def defaults(exchange_threshold=None, **kw) -> "PbtConfig":
        d = dict(pbt_period=5_000_000, mutate_fraction=0.70, mutation_rate=0.15,
                 mutation_factor=1.2, replace_fraction=0.30, window=100)
        d.update(kw)
        c = PbtConfig(**d)
        if exchange_threshold is not None:
            c.has_exchange_threshold = 1
            c.exchange_threshold = exchange_threshold
        return c


class AgentMeta(C.Structure):
    """AgentMeta (population.hpp:41-58)."""
    _fields_ = [("policy_id", C.c_uint32), ("n_reward_weights", C.c_int32),
                ("learning_rate", C.c_double), ("entropy_coef", C.c_double),
                ("adam_beta1", C.c_double),
                ("reward_weights", C.c_double * PBT_MAX_REWARD_WEIGHTS)]

    @staticmethod
    def make(learning_rate=1e-4, entropy_coef=0.003, adam_beta1=0.9, reward_weights=()):
        a = AgentMeta(0, len(reward_weights), learning_rate, entropy_coef, adam_beta1)
        for i, w in enumerate(reward_weights):
            a.reward_weights[i] = w
        return a

    def as_dict(self):
        return {"policy_id": self.policy_id, "learning_rate": self.learning_rate,
                "entropy_coef": self.entropy_coef, "adam_beta1": self.adam_beta1,
                "reward_weights": list(self.reward_weights[:self.n_reward_weights])}


class PbtEvent(C.Structure):
    _fields_ = [("frame", C.c_int64), ("agent", C.c_uint32), ("event", C.c_int32),
                ("field", C.c_char * 32), ("old_value", C.c_double), ("new_value", C.c_double)]

    def as_tuple(self):
        return (self.frame, self.agent, PBT_EVENTS[self.event], self.field.decode(),
                self.old_value, self.new_value)


PBT_COPY_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.c_uint32)


def params_copy(dst: "Context", src: "Context"):
    """dst learner takes src's parameters + Adam state and publishes them."""
    check(_L.appo_params_copy(dst.h, src.h))


class PbtController:
    """Population-based training over P learners (appo_pbt_*; population.hpp
    pbt_step + runner.hpp PbtController).  copy_weights: None, a list of
    learner Contexts (device-to-device copies), or a Python callable
    ``f(dst, src)``."""

    def __init__(self, cfg: PbtConfig, P: int, seed: int, init=None, copy_weights=None,
                 pipeline_seed: bool = False):
        if pipeline_seed:
            seed = int(_L.appo_pbt_controller_seed(seed))
        arr = None
        if init is not None:
            arr = (AgentMeta * P)(*init)
        h = C.c_void_p()
        check(_L.appo_pbt_create(C.byref(cfg), P, seed, arr, C.byref(h)))
        self.h, self.P = h, P
        self._set_copy(copy_weights)

    def _set_copy(self, copy_weights):
        self._user = None
        if copy_weights is None:
            self._fn = None
        elif isinstance(copy_weights, (list, tuple)):
            self._learners = list(copy_weights)
            self._user = (C.c_void_p * len(copy_weights))(*[c.h.value for c in copy_weights])
            self._fn = C.cast(_L.appo_pbt_copy_contexts, C.c_void_p)
        else:
            def tramp(_user, dst, src, f=copy_weights):
                try:
                    f(dst, src)
                    return 0
                except Exception:  # surfaced as a ContractError by the library
                    return 1
            self._cb = PBT_COPY_FN(tramp)
            self._fn = C.cast(self._cb, C.c_void_p)

    def close(self):
        if getattr(self, "h", None):
            _L.appo_pbt_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _events(self, buf, n):
        return [buf[i] for i in range(n)]

    def step(self, scores, frame: int):
        """One pbt_step; scores: list of float or None (exempt)."""
        sc = np.array([0.0 if s is None else float(s) for s in scores], dtype=np.float64)
        has = np.array([s is not None for s in scores], dtype=np.uint8)
        assert sc.size == self.P
        cap = int(_L.appo_pbt_max_events(self.h))
        buf = (PbtEvent * cap)()
        n = _i()
        check(_L.appo_pbt_step(self.h, sc.ctypes.data_as(C.c_void_p),
                               has.ctypes.data_as(C.c_void_p), frame, self._fn,
                               C.cast(self._user, C.c_void_p) if self._user else None, buf, cap,
                               C.byref(n)))
        return self._events(buf, n.value)

    def record(self, policy: int, value: float):
        check(_L.appo_pbt_record(self.h, policy, value))

    def score(self, policy: int):
        s, has = C.c_double(), _i()
        check(_L.appo_pbt_score(self.h, policy, C.byref(s), C.byref(has)))
        return s.value if has.value else None

    def tick(self, frames: int):
        """PbtController::tick: returns the events of a step, or None."""
        cap = int(_L.appo_pbt_max_events(self.h))
        buf = (PbtEvent * cap)()
        n, fired = _i(), _i()
        check(_L.appo_pbt_tick(self.h, frames, self._fn,
                               C.cast(self._user, C.c_void_p) if self._user else None, buf, cap,
                               C.byref(n), C.byref(fired)))
        return self._events(buf, n.value) if fired.value else None

    def agent(self, i: int) -> AgentMeta:
        a = AgentMeta()
        check(_L.appo_pbt_get_agent(self.h, i, C.byref(a)))
        return a

    def hparams(self, i: int, base: HParams | None = None) -> HParams:
        """Learner hyper-parameters of policy i (HyperBlock hand-back, runner.hpp:222-232)."""
        a = self.agent(i)
        hp = HParams.defaults() if base is None else HParams.from_buffer_copy(base)
        hp.lr, hp.entropy_coef, hp.beta1 = a.learning_rate, a.entropy_coef, a.adam_beta1
        return hp

    @staticmethod
    def format_events(events, header: bool = True) -> str:
        arr = (PbtEvent * max(1, len(events)))(*events)
        ln = _u64()
        check(_L.appo_pbt_format_events(arr, len(events), int(header), None, 0, C.byref(ln)))
        out = C.create_string_buffer(ln.value + 1)
        check(_L.appo_pbt_format_events(arr, len(events), int(header), out, ln.value + 1, None))
        return out.value.decode()


EPI_BIAS, EPI_ELU, EPI_DELU, EPI_BF16, EPI_TRANS, EPI_ACCUM = 1, 2, 4, 8, 16, 32

from .store import TrajectoryStore  # noqa: E402,F401

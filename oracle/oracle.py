"""ctypes bindings for the test oracles.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  The product package
(paper_2006_11751_b200) never imports it.

* ``Oracle``    -- oracle/liboracle.so, the fp64 C restatement (appo_oracle.c).
* ``Reference`` -- oracle/_ref/libappo_ref.so, the reference headers compiled
  unchanged (oracle/ref_shim.cpp); present wherever ``make -C oracle`` ran with
  /root/reference mounted, shipped prebuilt to the GPU box.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libappo_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")

# hyper-parameter vector layout shared with orc_learner_step
HP_KEYS = ["lr", "beta1", "beta2", "eps", "grad_clip", "entropy_coef", "value_coef",
           "clip_low", "clip_high", "rho_bar", "c_bar", "gamma", "adv_source", "normalize",
           "gae_lambda"]
HP_DEFAULT = dict(lr=1e-4, beta1=0.9, beta2=0.999, eps=1e-6, grad_clip=4.0,
                  entropy_coef=0.003, value_coef=0.5, clip_low=1.0 / 1.1, clip_high=1.1,
                  rho_bar=1.0, c_bar=1.0, gamma=0.99, adv_source=0, normalize=0,
                  gae_lambda=0.95)


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class Oracle:
    def __init__(self, path: str = LIB):
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.L = L
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_derive_seed.restype = C.c_uint64
        L.orc_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_uniform.restype = C.c_double
        L.orc_uniform.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_vtrace.restype = C.c_int
        L.orc_vtrace.argtypes = [C.c_int, _dp, _dp, C.c_double, _dp, _dp, _u8p, C.c_double,
                                 C.c_double, C.c_double, _dp, _dp, _dp, _dp]
        L.orc_nstep_returns.restype = None
        L.orc_nstep_returns.argtypes = [C.c_int, _dp, C.c_double, _u8p, C.c_double, _dp]
        L.orc_gae.restype = None
        L.orc_gae.argtypes = [C.c_int, _dp, _dp, C.c_double, _u8p, C.c_double, C.c_double, _dp,
                              _dp]
        L.orc_ppo_objective.restype = C.c_double
        L.orc_ppo_objective.argtypes = [C.c_double] * 4
        L.orc_ppo_dratio.restype = C.c_double
        L.orc_ppo_dratio.argtypes = [C.c_double] * 4
        L.orc_importance_ratio.restype = C.c_double
        L.orc_importance_ratio.argtypes = [C.c_double] * 2
        L.orc_total_loss.restype = C.c_int
        L.orc_total_loss.argtypes = [C.c_int, _dp, _dp, _dp, _dp, _dp, C.c_double, C.c_double,
                                     C.c_double, C.c_double, _dp]
        L.orc_softmax.restype = None
        L.orc_softmax.argtypes = [C.c_int, _dp, _dp]
        L.orc_sample.restype = C.c_int
        L.orc_sample.argtypes = [C.c_int, _dp, C.c_double, C.POINTER(C.c_double)]
        L.orc_logp_entropy.restype = C.c_int
        L.orc_logp_entropy.argtypes = [C.c_int, _dp, C.c_int, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]
        L.orc_adam_step.restype = C.c_int
        L.orc_adam_step.argtypes = [C.c_long, _dp, _dp, _dp, _dp, C.POINTER(C.c_long),
                                    C.c_double, C.c_double, C.c_double, C.c_double, C.c_double]
        L.orc_slot_offsets.restype = None
        L.orc_slot_offsets.argtypes = [C.c_uint32] * 4 + [C.c_int] * 4 + [_u64p]
        L.orc_gen_obs.restype = None
        L.orc_gen_obs.argtypes = [C.c_uint64, C.c_uint32, C.c_long, _u8p]
        L.orc_gen_reward.restype = C.c_double
        L.orc_gen_reward.argtypes = [C.c_uint64, C.c_uint32]
        L.orc_model_param_count.restype = C.c_long
        L.orc_model_param_count.argtypes = [C.c_int] * 4
        L.orc_model_init.restype = None
        L.orc_model_init.argtypes = [C.c_int] * 4 + [C.c_uint64, _dp]
        L.orc_policy_forward.restype = None
        L.orc_policy_forward.argtypes = [C.c_int] * 4 + [_dp, C.c_int, _u8p, _dp, _dp, _dp, _dp,
                                                         C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_learner_step.restype = C.c_int
        L.orc_learner_step.argtypes = ([C.c_int] * 4 + [_dp, _dp, _dp, C.POINTER(C.c_long),
                                                        C.c_int, C.c_int, _u8p, _dp, _i32p, _dp,
                                                        _dp, _u8p, _dp, C.c_int, _dp, _dp,
                                                        C.c_void_p, C.c_void_p, C.c_void_p,
                                                        C.c_void_p])

    # -- off-policy -------------------------------------------------------
    def vtrace(self, rewards, values, bootstrap, tlogp, blogp, dones, rho_bar=1.0, c_bar=1.0,
               gamma=0.99):
        r = _c(rewards, np.float64)
        T = r.shape[0]
        outs = [np.zeros(T) for _ in range(4)]
        st = self.L.orc_vtrace(T, r, _c(values, np.float64), float(bootstrap),
                               _c(tlogp, np.float64), _c(blogp, np.float64),
                               _c(dones, np.uint8), rho_bar, c_bar, gamma, *outs)
        return st, outs

    def vtrace_batch(self, rewards, values, boot, tlogp, blogp, dones, rho_bar=1.0, c_bar=1.0,
                     gamma=0.99):
        n, T = rewards.shape
        v = np.zeros((n, T)); pg = np.zeros((n, T)); rho = np.zeros((n, T)); c = np.zeros((n, T))
        for i in range(n):
            st, (a, b, cc, d) = self.vtrace(rewards[i], values[i], boot[i], tlogp[i], blogp[i],
                                            dones[i], rho_bar, c_bar, gamma)
            if st:
                return st, None
            v[i], pg[i], rho[i], c[i] = a, b, cc, d
        return 0, (v, pg, rho, c)

    def nstep_returns(self, rewards, bootstrap, dones, gamma):
        r = _c(rewards, np.float64)
        out = np.zeros(r.shape[0])
        self.L.orc_nstep_returns(r.shape[0], r, float(bootstrap), _c(dones, np.uint8), gamma, out)
        return out

    def gae(self, rewards, values, bootstrap, dones, gamma, lam):
        r = _c(rewards, np.float64)
        adv = np.zeros(r.shape[0]); ret = np.zeros(r.shape[0])
        self.L.orc_gae(r.shape[0], r, _c(values, np.float64), float(bootstrap),
                       _c(dones, np.uint8), gamma, lam, adv, ret)
        return adv, ret

    def total_loss(self, ratios, adv, values, vt, ent, lo=1 / 1.1, hi=1.1, vc=0.5, ec=0.003):
        out = np.zeros(4)
        n = len(ratios)
        st = self.L.orc_total_loss(n, _c(ratios, np.float64), _c(adv, np.float64),
                                   _c(values, np.float64), _c(vt, np.float64),
                                   _c(ent, np.float64), lo, hi, vc, ec, out)
        return st, out

    def softmax(self, logits):
        lg = _c(logits, np.float64)
        p = np.zeros_like(lg)
        self.L.orc_softmax(lg.shape[0], lg, p)
        return p

    def logp_entropy(self, logits, action):
        lg = _c(logits, np.float64)
        lp, e = C.c_double(), C.c_double()
        st = self.L.orc_logp_entropy(lg.shape[0], lg, int(action), C.byref(lp), C.byref(e))
        return st, lp.value, e.value

    def sample(self, logits, u):
        lg = _c(logits, np.float64)
        lp = C.c_double()
        a = self.L.orc_sample(lg.shape[0], lg, float(u), C.byref(lp))
        return a, lp.value

    def adam_step(self, theta, m, v, g, t, lr=1e-4, b1=0.9, b2=0.999, eps=1e-6, clip=4.0):
        tt = C.c_long(t)
        st = self.L.orc_adam_step(theta.shape[0], theta, m, v, _c(g, np.float64), C.byref(tt),
                                  lr, b1, b2, eps, clip)
        return st, tt.value

    def slot_offsets(self, T, obs_dim, hidden_dim, n_heads, elems=(1, 4, 4, 4)):
        out = np.zeros(10, dtype=np.uint64)
        self.L.orc_slot_offsets(T, obs_dim, hidden_dim, n_heads, *elems, out)
        return [int(x) for x in out]

    def gen_obs(self, env_seed, step, obs_dim):
        out = np.zeros(obs_dim, dtype=np.uint8)
        self.L.orc_gen_obs(env_seed, step, obs_dim, out)
        return out

    # -- model ------------------------------------------------------------
    def param_count(self, C_, H, W, A):
        return self.L.orc_model_param_count(C_, H, W, A)

    def init_params(self, C_, H, W, A, seed):
        th = np.zeros(self.param_count(C_, H, W, A))
        self.L.orc_model_init(C_, H, W, A, seed, th)
        return th

    def policy_forward(self, shape, theta, obs, h_in, u=None):
        C_, H, W, A = shape
        B = obs.shape[0]
        obs = _c(obs.reshape(B, -1), np.uint8)
        h_out = np.zeros((B, 512)); logits = np.zeros((B, A)); values = np.zeros(B)
        actions = np.zeros(B, dtype=np.int32); logp = np.zeros(B)
        if u is not None:
            u = _c(u, np.float64)
            self.L.orc_policy_forward(C_, H, W, A, _c(theta, np.float64), B, obs,
                                      _c(h_in, np.float64), h_out, logits, values,
                                      u.ctypes.data, actions.ctypes.data, logp.ctypes.data)
        else:
            self.L.orc_policy_forward(C_, H, W, A, _c(theta, np.float64), B, obs,
                                      _c(h_in, np.float64), h_out, logits, values, None, None,
                                      None)
        return dict(h_out=h_out, logits=logits, values=values, actions=actions, logp=logp)

    def learner_step(self, shape, theta, m, v, t, obs, h0, actions, blogp, rewards, dones,
                     hp=None, do_adam=True):
        """obs: [n_traj, T+1, C*H*W] u8 (index T = bootstrap obs)."""
        C_, H, W, A = shape
        hpd = dict(HP_DEFAULT)
        hpd.update(hp or {})
        hpv = np.array([float(hpd[k]) for k in HP_KEYS])
        n_traj, T1 = obs.shape[0], obs.shape[1]
        T = T1 - 1
        P = theta.shape[0]
        grad = np.zeros(P); stats = np.zeros(8)
        B = n_traj * T
        vt = np.zeros(B); adv = np.zeros(B); vals = np.zeros(B); tl = np.zeros(B)
        tt = C.c_long(t)
        st = self.L.orc_learner_step(C_, H, W, A, theta, m, v, C.byref(tt), n_traj, T,
                                     _c(obs.reshape(n_traj * T1, -1), np.uint8),
                                     _c(h0, np.float64), _c(actions, np.int32),
                                     _c(blogp, np.float64), _c(rewards, np.float64),
                                     _c(dones, np.uint8), hpv, int(do_adam), grad, stats,
                                     vt.ctypes.data, adv.ctypes.data, vals.ctypes.data,
                                     tl.ctypes.data)
        return dict(status=st, grad=grad, stats=stats, v_targets=vt, adv=adv, values=vals,
                    tlogp=tl, t=tt.value)


class Reference:
    """The reference headers compiled unchanged (oracle/_ref/libappo_ref.so)."""

    def save_checkpoint_mlp(self, path, obs_dim, trunk, heads, seed, version, t):
        """save_checkpoint (policy.hpp:545-564) of an init_params MLP; returns n."""
        h = np.ascontiguousarray(heads, dtype=np.int32)
        return int(self.L.ref_save_checkpoint_mlp(os.fsencode(path), obs_dim, trunk, h, len(h),
                                                  seed, version, t))

    def spec_hash_mlp(self, obs_dim, hidden, trunk, heads):
        h = np.ascontiguousarray(heads, dtype=np.int32)
        return int(self.L.ref_spec_hash_mlp(obs_dim, hidden, trunk, h, len(h)))

    def __init__(self, path: str = REF_LIB):
        L = C.CDLL(path)
        self.L = L
        L.ref_save_checkpoint_mlp.restype = C.c_longlong
        L.ref_save_checkpoint_mlp.argtypes = [C.c_char_p, C.c_int, C.c_int, _i32p, C.c_int,
                                              C.c_uint64, C.c_longlong, C.c_longlong]
        L.ref_spec_hash_mlp.restype = C.c_uint64
        L.ref_fnv1a64.restype = C.c_uint64
        L.ref_fnv1a64.argtypes = [C.c_char_p, C.c_size_t]
        L.ref_spec_hash_mlp.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, C.c_int]
        L.ref_vtrace.restype = C.c_int
        L.ref_vtrace.argtypes = [C.c_int, _dp, _dp, C.c_double, _dp, _dp, _u8p, C.c_double,
                                 C.c_double, C.c_double, _dp, _dp, _dp, _dp]
        L.ref_vtrace_range.restype = C.c_int
        L.ref_vtrace_range.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp, _u8p,
                                       C.c_double, C.c_double, C.c_double, _dp, _dp]
        L.ref_nstep_returns.restype = None
        L.ref_nstep_returns.argtypes = [C.c_int, _dp, C.c_double, _u8p, C.c_double, _dp]
        L.ref_ppo_objective.restype = C.c_double
        L.ref_ppo_objective.argtypes = [C.c_double] * 4
        L.ref_ppo_dratio.restype = C.c_double
        L.ref_ppo_dratio.argtypes = [C.c_double] * 4
        L.ref_importance_ratio.restype = C.c_double
        L.ref_importance_ratio.argtypes = [C.c_double] * 2
        L.ref_total_loss.restype = C.c_int
        L.ref_total_loss.argtypes = [C.c_int, _dp, _dp, _dp, _dp, _dp, C.c_double, C.c_double,
                                     C.c_double, C.c_double, _dp]
        L.ref_softmax.restype = None
        L.ref_softmax.argtypes = [C.c_int, _dp, _dp]
        L.ref_log_prob_entropy.restype = C.c_int
        L.ref_log_prob_entropy.argtypes = [C.c_int, _dp, C.c_int, C.POINTER(C.c_double),
                                           C.POINTER(C.c_double)]
        L.ref_sample_actions.restype = None
        L.ref_sample_actions.argtypes = [C.c_int, _dp, C.c_uint64, C.c_int, _i32p, _dp]
        L.ref_optimizer_step.restype = C.c_int
        L.ref_optimizer_step.argtypes = [C.c_long, _dp, _dp, _dp, _dp, C.POINTER(C.c_long),
                                         C.c_double, C.c_double, C.c_double, C.c_double,
                                         C.c_double]
        L.ref_slot_offsets.restype = None
        L.ref_slot_offsets.argtypes = [C.c_uint32] * 4 + [_u64p]
        L.ref_rng_new.restype = C.c_void_p
        L.ref_rng_new.argtypes = [C.c_uint64]
        L.ref_rng_free.restype = None
        L.ref_rng_free.argtypes = [C.c_void_p]
        L.ref_random_instance.restype = None
        L.ref_random_instance.argtypes = [C.c_void_p, C.c_int, C.c_double, _dp, _dp, _dp, _dp,
                                          _u8p, _dp]
        L.ref_splitmix64.restype = C.c_uint64
        L.ref_splitmix64.argtypes = [C.c_uint64]
        L.ref_derive_seed.restype = C.c_uint64
        L.ref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]

    def ppo_grads_injected(self, logits, values, actions, blogp, adv, vt, lo=1 / 1.1, hi=1.1,
                           vc=0.5, ec=0.003):
        """compute_gradients with injected logits/values (ref_shim.cpp): per-sample
        dlogits [n][A] and dL/dV [n] of the batch-mean loss, loss4, mean ratio."""
        lg = _c(logits, np.float64)
        n, A = lg.shape
        dl = np.zeros((n, A)); dv = np.zeros(n); loss = np.zeros(4); mr = C.c_double()
        L = self.L
        L.ref_ppo_grads_injected.restype = C.c_int
        L.ref_ppo_grads_injected.argtypes = [C.c_int, C.c_int, _dp, _dp, _i32p, _dp, _dp, _dp,
                                             C.c_double, C.c_double, C.c_double, C.c_double,
                                             _dp, _dp, _dp, C.POINTER(C.c_double)]
        st = L.ref_ppo_grads_injected(n, A, lg, _c(values, np.float64), _c(actions, np.int32),
                                      _c(blogp, np.float64), _c(adv, np.float64),
                                      _c(vt, np.float64), lo, hi, vc, ec, dl, dv, loss,
                                      C.byref(mr))
        return st, dict(dlogits=dl, dv=dv, loss=loss, mean_ratio=mr.value)

    def logp_entropy_heads(self, sizes, logits, actions):
        """log_prob_and_entropy (policy.hpp:262-281) over factored heads."""
        sz = _c(sizes, np.int32)
        lg = _c(logits, np.float64)
        B = lg.shape[0]
        act = _c(actions, np.int32)
        lp = np.zeros(B); en = np.zeros(B)
        L = self.L
        L.ref_log_prob_entropy_heads.restype = C.c_int
        L.ref_log_prob_entropy_heads.argtypes = [C.c_int, _i32p, C.c_int, _dp, _i32p, _dp, _dp]
        st = L.ref_log_prob_entropy_heads(len(sz), sz, B, lg, act, lp, en)
        return st, lp, en

    def mlp_stand_in_time(self, obs_dim=27648, trunk=512, A=6, B=8, reps=2):
        """The reference's MLP stand-in at the Doom input through its own
        forward_batch / compute_gradients / optimizer_step on one thread
        (ref_shim.cpp): seconds per sample (forward, gradient), per Adam call."""
        L = self.L
        L.ref_mlp_stand_in_time.restype = C.c_int
        L.ref_mlp_stand_in_time.argtypes = [C.c_int] * 5 + [_dp]
        out = np.zeros(4)
        st = L.ref_mlp_stand_in_time(obs_dim, trunk, A, B, reps, out)
        return st, dict(forward_s_per_sample=out[0], gradient_s_per_sample=out[1],
                        optimizer_s=out[2], n_params=int(out[3]))

    def dump_trajectory(self, path, obs, hidden, actions, rewards, logp, dones, versions,
                        boot_obs, boot_hidden, env=0, worker=0, policy=0):
        """dump_trajectory (trajstore.hpp:335-359) of a slot the reference itself
        filled with begin / write_step / set_bootstrap (ref_shim.cpp); returns
        the guarded status (0 ok, 1 contract, 3 numeric)."""
        obs = _c(obs, np.float64)
        T, od = obs.shape
        hid = _c(hidden, np.float64)
        L = self.L
        L.ref_dump_trajectory.restype = C.c_int
        L.ref_dump_trajectory.argtypes = [C.c_uint32] * 3 + [_dp, _dp, _i32p, _dp, _dp, _u8p,
                                          C.POINTER(C.c_int64), _dp, _dp] + \
            [C.c_uint32] * 3 + [C.c_char_p]
        ver = _c(versions, np.int64)
        return int(L.ref_dump_trajectory(T, od, hid.shape[1], obs, hid, _c(actions, np.int32),
                                         _c(rewards, np.float64), _c(logp, np.float64),
                                         _c(dones, np.uint8),
                                         ver.ctypes.data_as(C.POINTER(C.c_int64)),
                                         _c(boot_obs, np.float64), _c(boot_hidden, np.float64),
                                         env, worker, policy, os.fsencode(path)))

    @staticmethod
    def available(path: str = REF_LIB) -> bool:
        return os.path.exists(path)

    def vtrace(self, rewards, values, bootstrap, tlogp, blogp, dones, rho_bar=1.0, c_bar=1.0,
               gamma=0.99):
        r = _c(rewards, np.float64)
        T = r.shape[0]
        outs = [np.zeros(T) for _ in range(4)]
        st = self.L.ref_vtrace(T, r, _c(values, np.float64), float(bootstrap),
                               _c(tlogp, np.float64), _c(blogp, np.float64),
                               _c(dones, np.uint8), rho_bar, c_bar, gamma, *outs)
        return st, outs

    def nstep_returns(self, rewards, bootstrap, dones, gamma):
        r = _c(rewards, np.float64)
        out = np.zeros(r.shape[0])
        self.L.ref_nstep_returns(r.shape[0], r, float(bootstrap), _c(dones, np.uint8), gamma,
                                 out)
        return out

    def total_loss(self, ratios, adv, values, vt, ent, lo=1 / 1.1, hi=1.1, vc=0.5, ec=0.003):
        out = np.zeros(4)
        st = self.L.ref_total_loss(len(ratios), _c(ratios, np.float64), _c(adv, np.float64),
                                   _c(values, np.float64), _c(vt, np.float64),
                                   _c(ent, np.float64), lo, hi, vc, ec, out)
        return st, out

    def softmax(self, logits):
        lg = _c(logits, np.float64)
        p = np.zeros_like(lg)
        self.L.ref_softmax(lg.shape[0], lg, p)
        return p

    def logp_entropy(self, logits, action):
        lg = _c(logits, np.float64)
        lp, e = C.c_double(), C.c_double()
        st = self.L.ref_log_prob_entropy(lg.shape[0], lg, int(action), C.byref(lp), C.byref(e))
        return st, lp.value, e.value

    def sample_actions(self, logits, seed, count):
        lg = _c(logits, np.float64)
        a = np.zeros(count, dtype=np.int32); lp = np.zeros(count)
        self.L.ref_sample_actions(lg.shape[0], lg, seed, count, a, lp)
        return a, lp

    def optimizer_step(self, theta, m, v, g, t, lr=1e-4, b1=0.9, b2=0.999, eps=1e-6, clip=4.0):
        tt = C.c_long(t)
        st = self.L.ref_optimizer_step(theta.shape[0], theta, m, v, _c(g, np.float64),
                                       C.byref(tt), lr, b1, b2, eps, clip)
        return st, tt.value

    def slot_offsets(self, T, obs_dim, hidden_dim, n_heads):
        out = np.zeros(10, dtype=np.uint64)
        self.L.ref_slot_offsets(T, obs_dim, hidden_dim, n_heads, out)
        return [int(x) for x in out]

    def random_instances(self, seed, Ts, done_prob=0.15):
        """Yields instances exactly as acceptance.cpp:42-56 draws them."""
        st = self.L.ref_rng_new(seed)
        try:
            out = []
            for T in Ts:
                r = np.zeros(T); v = np.zeros(T); tl = np.zeros(T); bl = np.zeros(T)
                d = np.zeros(T, dtype=np.uint8); b = np.zeros(1)
                self.L.ref_random_instance(st, T, done_prob, r, v, tl, bl, d, b)
                out.append(dict(rewards=r, values=v, tlogp=tl, blogp=bl, dones=d,
                                bootstrap=float(b[0])))
            return out
        finally:
            self.L.ref_rng_free(st)

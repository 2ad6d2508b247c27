"""Device-resident trajectory store: ``n_slots`` fixed-shape slots of layout v2
in one HBM region (replaces TrajectoryStore / SlotRegion, trajstore.hpp:236-261,
transport.hpp:399-460, whose slots live in shared host memory).

Layout v2 keeps the reference's 64-byte in-slot header, field order and align8
offsets algorithm (trajstore.hpp:41-87, docs/shared_memory_layout.md:23-51) with
device element types: obs u8, hidden f32, actions i32, rewards f32, logp f32,
dones u8, versions i64, boot_obs u8, boot_hidden f32.  ``to_reference_dump``
exports a slot in the reference's dump format (trajstore.hpp:335-359) with
f64 arrays, for byte comparison with ``dump_trajectory``.
"""
from __future__ import annotations

import struct

import numpy as np


class TrajectoryStore:
    def __init__(self, desc, n_slots: int, device: int = 0):
        import torch
        from . import slot_layout
        self.torch = torch
        self.desc = desc
        self.layout = slot_layout(desc)
        # slot stride: the layout-v2 slot rounded up to 16 B (vector loads need
        # 16-byte aligned slot bases); at the Doom shape it is exactly the
        # reference's dense stride (980,704 B).  The in-slot byte layout is
        # exactly trajstore.hpp's Offsets algorithm.
        self.slot_bytes = (self.layout["total"] + 15) // 16 * 16
        self.n_slots = n_slots
        self.T = desc.T
        self.obs_dim = desc.obs_dim
        # device = "cpu": a host region (layout / dump tests without a GPU; the
        # library's kernels only ever see device regions)
        dev = "cpu" if device == "cpu" else f"cuda:{device}"
        self.region = torch.zeros(n_slots * self.slot_bytes, dtype=torch.uint8, device=dev)
        # the region is written by library streams other than torch's: make the
        # zero fill visible to them before first use
        if dev != "cpu":
            torch.cuda.synchronize(device)

    # ---- typed views of one slot (device tensors aliasing the region) ----
    def _view(self, slot: int, field: str, dtype, count: int):
        torch = self.torch
        o = slot * self.slot_bytes + self.layout[field]
        nbytes = count * torch.empty(0, dtype=dtype).element_size()
        return self.region[o:o + nbytes].view(dtype)

    def obs(self, slot):
        return self._view(slot, "obs", self.torch.uint8, self.T * self.obs_dim).view(self.T, -1)

    def hidden(self, slot):
        return self._view(slot, "hidden", self.torch.float32, self.T * 512).view(self.T, 512)

    def actions(self, slot):
        return self._view(slot, "actions", self.torch.int32, self.T)

    def rewards(self, slot):
        return self._view(slot, "rewards", self.torch.float32, self.T)

    def logp(self, slot):
        return self._view(slot, "logp", self.torch.float32, self.T)

    def dones(self, slot):
        return self._view(slot, "dones", self.torch.uint8, self.T)

    def versions(self, slot):
        return self._view(slot, "versions", self.torch.int64, self.T)

    def boot_obs(self, slot):
        return self._view(slot, "boot_obs", self.torch.uint8, self.obs_dim)

    def boot_hidden(self, slot):
        return self._view(slot, "boot_hidden", self.torch.float32, 512)

    def header(self, slot):
        return self.region[slot * self.slot_bytes: slot * self.slot_bytes + 64]

    def write_slot(self, slot: int, obs, h0, actions, rewards, logp, dones, versions=None,
                   boot_obs=None, boot_hidden=None, env_id=0, worker_id=0, policy_id=0):
        """Host-side fill of one complete slot (test / staging helper).  Enforces
        the write_step contracts of trajstore.hpp:166-189 on the whole record."""
        torch = self.torch
        T = self.T
        from . import ContractError, NumericError
        logp = np.asarray(logp, np.float32)
        if np.any(logp > 1e-6):
            raise ContractError("write_step: behavior log-prob above zero")
        versions = np.zeros(T, np.int64) if versions is None else np.asarray(versions, np.int64)
        if np.any(np.diff(versions) < 0):
            raise ContractError("write_step: policy_version must be non-decreasing")
        obs = np.asarray(obs, np.uint8).reshape(T, -1)
        if obs.shape[1] != self.obs_dim:
            raise ContractError("write_step: obs dim mismatch")
        if not np.all(np.isfinite(np.asarray(rewards, np.float32))):
            raise NumericError("write_step: non-finite reward")
        dev = self.region.device
        self.obs(slot).copy_(torch.from_numpy(obs).to(dev))
        hid = np.zeros((T, 512), np.float32)
        hid[0] = np.asarray(h0, np.float32)
        self.hidden(slot).copy_(torch.from_numpy(hid).to(dev))
        self.actions(slot).copy_(torch.from_numpy(np.asarray(actions, np.int32)).to(dev))
        self.rewards(slot).copy_(torch.from_numpy(np.asarray(rewards, np.float32)).to(dev))
        self.logp(slot).copy_(torch.from_numpy(logp).to(dev))
        self.dones(slot).copy_(torch.from_numpy(np.asarray(dones, np.uint8)).to(dev))
        self.versions(slot).copy_(torch.from_numpy(versions).to(dev))
        if boot_obs is not None:
            self.boot_obs(slot).copy_(torch.from_numpy(np.asarray(boot_obs, np.uint8)).to(dev))
        if boot_hidden is not None:
            self.boot_hidden(slot).copy_(
                torch.from_numpy(np.asarray(boot_hidden, np.float32)).to(dev))
        hdr = struct.pack("<10I", T, self.obs_dim, 512, 1, T, env_id, worker_id, policy_id, 0, 1)
        self.header(slot)[:40].copy_(torch.frombuffer(bytearray(hdr), dtype=torch.uint8).to(dev))

    def to_reference_dump(self, slot: int) -> bytes:
        """Dump in the reference format (trajstore.hpp:335-359): 32-byte header
        {T, obs_dim, hidden_dim, n_heads, 0...}, then the packed arrays with the
        reference's element types (f64 obs/hidden/rewards/logp/boot arrays)."""
        T, od = self.T, self.obs_dim
        raw = self.region[slot * self.slot_bytes:(slot + 1) * self.slot_bytes].cpu().numpy()
        L = self.layout
        g = lambda f, dt, n: np.frombuffer(raw[L[f]:L[f] + n * np.dtype(dt).itemsize], dt)
        parts = [struct.pack("<8I", T, od, 512, 1, 0, 0, 0, 0),
                 g("obs", np.uint8, T * od).astype(np.float64).tobytes(),
                 g("hidden", np.float32, T * 512).astype(np.float64).tobytes(),
                 g("actions", np.int32, T).tobytes(),
                 g("rewards", np.float32, T).astype(np.float64).tobytes(),
                 g("logp", np.float32, T).astype(np.float64).tobytes(),
                 g("dones", np.uint8, T).tobytes(),
                 g("versions", np.int64, T).tobytes(),
                 g("boot_obs", np.uint8, od).astype(np.float64).tobytes(),
                 g("boot_hidden", np.float32, 512).astype(np.float64).tobytes()]
        return b"".join(parts)

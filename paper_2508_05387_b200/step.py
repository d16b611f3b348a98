"""One learner step on one rank, driven through the C ABI (the public API a trainer's ``step()`` calls).

    h2d        rollouts of this rank's shard, host (pinned) -> device
    pack       echo_pack_batch                 (1) lag filter + pack; one 32-byte D2H read sizes the logits
    advantage  echo_group_advantage            (2) GRPO advantage
    stats1     all-reduce {N, advantage/reward sums, group counts} -> N_global stays on the device
    rebalance  (f3, optional) move whole kept rollouts between ranks so every rank holds ~N_global / W tokens:
               NCCL all-to-all of the packed arrays, echo_csr_from_lengths rebuilds the CSR
    loss       echo_policy_loss_fwd_bwd        (3)-(5) once per micro-batch of logits rows (in place)
    finish     echo_loss_stats + all-reduce    statistics of the step, read back for logging

torch is used for device memory, pinned host staging, streams and process groups only.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import abi
from .parallel import allreduce_sum_, exchange, reduce_loss_stats_, reshard_plan, LOSS_STATS, STATS1


@dataclass
class PackInfo:
    status: int
    first_bad_rollout: int
    n_groups_kept: int
    n_rollouts_kept: int
    n_tokens: int


class LearnerStep:
    def __init__(self, *, n_rollouts: int, group_size: int, max_len: int, vocab: int, dtype: str = "bf16",
                 has_ref: bool = True, device=None, group=None, eps: float = 1e-8):
        self.R, self.G, self.S, self.V = n_rollouts, group_size, max_len, vocab
        self.dtype = dtype
        self.edtype = abi.ECHO_BF16 if dtype == "bf16" else abi.ECHO_F32
        self.has_ref = has_ref
        self.eps = eps
        self.group = group
        self.launches = 0
        dev = torch.device("cuda") if device is None else torch.device(device)
        self.device = dev
        R, S = n_rollouts, max_len
        cap = max(R * S, 1)
        e = dict(device=dev)
        # inputs
        self.version = torch.empty(R, dtype=torch.int64, **e)
        self.resp_len = torch.empty(R, dtype=torch.int32, **e)
        self.reward = torch.empty(R, dtype=torch.float32, **e)
        self.action = torch.empty(R * S, dtype=torch.int32, **e)
        self.old_logp = torch.empty(R * S, dtype=torch.float32, **e)
        self.ref_logp = torch.empty(R * S, dtype=torch.float32, **e) if has_ref else None
        # packed state
        self.cap = cap
        self.kept_rollout = torch.empty(max(R, 1), dtype=torch.int32, **e)
        self.kept_offset = torch.empty(R + 1, dtype=torch.int64, **e)
        self.tok_slot = torch.empty(cap, dtype=torch.int32, **e)
        self.tok_action = torch.empty(cap, dtype=torch.int32, **e)
        self.tok_old = torch.empty(cap, dtype=torch.float32, **e)
        self.tok_ref = torch.empty(cap, dtype=torch.float32, **e) if has_ref else None
        self.pack_result = torch.zeros(abi.PACK_RESULT_BYTES, dtype=torch.uint8, **e)
        self.adv_slot = torch.empty(max(R, 1), dtype=torch.float32, **e)
        self.adv_stats = torch.empty(6, dtype=torch.float64, **e)
        self.stats1 = torch.zeros(len(STATS1), dtype=torch.float64, **e)
        # per-token outputs
        self.tok_logp = torch.empty(cap, dtype=torch.float32, **e)
        self.tok_loss = torch.empty(cap, dtype=torch.float32, **e)
        self.tok_flags = torch.empty(cap, dtype=torch.uint8, **e)
        self.ws = torch.empty(abi.echo_loss_stats_workspace_bytes() // 8, dtype=torch.float64, **e)
        self.loss_stats = torch.empty(len(LOSS_STATS), dtype=torch.float64, **e)
        # pinned host staging for the two reads of a step
        self._packed = {k: getattr(self, k) for k in ("kept_rollout", "kept_offset", "tok_slot", "tok_action", "tok_old",
                                                       "tok_ref", "adv_slot")}   # rebalance() swaps these
        self._cap0 = cap
        self._rebalanced = False
        self.pack_host = torch.empty(abi.PACK_RESULT_BYTES, dtype=torch.uint8, pin_memory=True)
        self.stats_host = torch.empty(len(STATS1) + len(LOSS_STATS), dtype=torch.float64, pin_memory=True)
        self.pack_info: PackInfo | None = None

    # ------------------------------------------------------------------ inputs
    def h2d(self, version, resp_len, reward, action, old_logp, ref_logp=None) -> int:
        """Copy this step's rollouts (host tensors, ideally pinned) to the device; returns bytes moved."""
        n = 0
        for dst, src in ((self.version, version), (self.resp_len, resp_len), (self.reward, reward),
                         (self.action, action), (self.old_logp, old_logp), (self.ref_logp, ref_logp)):
            if dst is None or src is None:
                continue
            src = src.reshape(-1)
            dst[: src.numel()].copy_(src, non_blocking=True)
            n += src.numel() * src.element_size()
        return n

    # ------------------------------------------------------------------ (1) + (2)
    def pack(self, *, t_train: int, max_lag: int, rollout_base: int = 0, n_rollouts: int | None = None,
             read_back: bool = True, filter_mode: int = 0) -> PackInfo | None:
        """(1): filter_mode abi.ECHO_FILTER_GROUP (whole groups, uniform versions) or ECHO_FILTER_ROLLOUT (f3:
        per-rollout staleness filter; partial groups are normalised over their survivors in advantage())."""
        R = self.R if n_rollouts is None else n_rollouts
        if self._rebalanced:                       # undo a previous step's rebalance()
            for k, v in self._packed.items():
                setattr(self, k, v)
            self.cap = self._cap0
            self._rebalanced = False
        abi.echo_pack_batch_v2(R, self.G, self.S, self.V, t_train, max_lag, rollout_base, self.version, self.resp_len,
                               self.action, self.old_logp, self.ref_logp, self.cap, self.kept_rollout,
                               self.kept_offset, self.tok_slot, self.tok_action, self.tok_old, self.tok_ref,
                               self.pack_result, filter_mode)
        self.launches += abi.LAUNCHES["echo_pack_batch"]
        self._R_step, self._base = R, rollout_base
        if not read_back:
            return None
        self.pack_host.copy_(self.pack_result, non_blocking=True)
        torch.cuda.current_stream().synchronize()          # the step's one host sync: sizes the logits
        self.pack_info = PackInfo(**abi.parse_pack_result(bytes(self.pack_host.numpy().tobytes())))
        return self.pack_info

    def advantage(self):
        abi.echo_group_advantage(self._R_step, self.G, self.eps, self.reward, self.kept_rollout, self._base,
                                 self.pack_result, self.adv_slot, self.adv_stats)
        self.launches += abi.LAUNCHES["echo_group_advantage"]

    def reduce_counts(self) -> torch.Tensor:
        """stats1 = {N, sum A, sum A^2, sum r, sum r^2, n_zero_std, n_rollouts_kept, n_groups_kept, n_dropped},
        all-reduced; returns the device view holding N_global (fed to the loss kernel without a host sync)."""
        info = self.pack_info
        n_groups = self._R_step // self.G
        self.stats1[0] = float(info.n_tokens)
        self.stats1[1:7].copy_(self.adv_stats)
        self.stats1[7] = float(info.n_groups_kept)
        self.stats1[8] = float(n_groups - info.n_groups_kept)
        allreduce_sum_(self.stats1, self.group)
        return self.stats1[0:1]

    # ------------------------------------------------------------------ f3
    def rebalance(self, extra_tokens=()) -> dict:
        """Token-balanced resharding after the stale filter (call after reduce_counts).

        Every rank's kept rollouts form a contiguous block of the global kept sequence (rank-major = group order);
        ``parallel.reshard_plan`` splits that sequence into W contiguous ranges of ~N_global / W tokens and the
        packed per-rollout (global id, advantage, length) and per-token (action, old, ref) arrays move there with
        one all-to-all each.  The receiver rebuilds kept_offset / tok_slot with echo_csr_from_lengths.  Returns the
        plan (tokens per rank before and after; ``plan["extra"]`` holds the rebalanced ``extra_tokens``, e.g. the
        packed per-token advantages of PPO-GAE or per-token weights).  One host sync (the kept rollouts' lengths)."""
        import numpy as np
        import torch.distributed as dist
        info = self.pack_info
        n_r, n_t = info.n_rollouts_kept, info.n_tokens
        if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(self.group) == 1:
            return {"tokens_before": [n_t], "tokens_after": [n_t], "extra": [t[:n_t] for t in extra_tokens]}
        world, rank = dist.get_world_size(self.group), dist.get_rank(self.group)
        off = self.kept_offset[: n_r + 1].cpu().numpy()
        lens = np.diff(off).astype(np.int32)
        gathered = [None] * world
        dist.all_gather_object(gathered, lens, group=self.group)
        counts = [len(x) for x in gathered]
        plan = reshard_plan(counts, np.concatenate(gathered), world, rank)
        lens_d = torch.from_numpy(lens).to(self.device)
        kept_rollout, adv_slot, lens_r = exchange([self.kept_rollout[:n_r], self.adv_slot[:n_r], lens_d],
                                                  plan["send_rollouts"], plan["recv_rollouts"], self.group)
        tok = [self.tok_action[:n_t], self.tok_old[:n_t]] + ([self.tok_ref[:n_t]] if self.tok_ref is not None else [])
        extra = [t[:n_t] for t in extra_tokens]
        tok = exchange(tok + extra, plan["send_tokens"], plan["recv_tokens"], self.group)
        plan["extra"] = tok[len(tok) - len(extra):]
        tok = tok[: len(tok) - len(extra)]
        new_r, new_t = sum(plan["recv_rollouts"]), sum(plan["recv_tokens"])
        kept_offset = torch.empty(new_r + 1, dtype=torch.int64, device=self.device)
        tok_slot = torch.empty(max(new_t, 1), dtype=torch.int32, device=self.device)
        abi.echo_csr_from_lengths(new_r, lens_r, kept_offset, tok_slot)
        self.launches += abi.LAUNCHES["echo_csr_from_lengths"]
        self._rebalanced = True
        self.kept_rollout, self.adv_slot, self.kept_offset, self.tok_slot = kept_rollout, adv_slot, kept_offset, tok_slot
        self.tok_action, self.tok_old = tok[0], tok[1]
        self.tok_ref = tok[2] if self.tok_ref is not None else None
        if new_t > self.tok_logp.numel():            # per-token outputs sized for the new share
            e = dict(device=self.device)
            self.tok_logp = torch.empty(new_t, dtype=torch.float32, **e)
            self.tok_loss = torch.empty(new_t, dtype=torch.float32, **e)
            self.tok_flags = torch.empty(new_t, dtype=torch.uint8, **e)
        self.pack_info = PackInfo(info.status, info.first_bad_rollout, info.n_groups_kept, new_r, new_t)
        return plan

    def staleness_histogram(self, *, t_train: int, max_lag: int, n_bins: int = 8, n_rollouts: int | None = None,
                            reduce: bool = True, filter_mode: int = 0) -> torch.Tensor:
        """f3: this step's staleness histogram (echo_staleness_histogram; int64 [4, n_bins + 2]: kept / dropped
        rollouts and tokens per lag bin), summed over the ranks of the process group (NCCL all-reduce)."""
        R = self.R if n_rollouts is None else n_rollouts
        h = torch.empty(4, n_bins + 2, dtype=torch.int64, device=self.device)
        abi.echo_staleness_histogram(R, self.G, self.S, t_train, max_lag, self.version, self.resp_len, n_bins, h,
                                     filter_mode)
        self.launches += abi.LAUNCHES["echo_staleness_histogram"]
        if reduce:
            allreduce_sum_(h, self.group)
        return h

    # ------------------------------------------------------------------ f2
    def token_logp_from_hidden(self, hidden, weight, out=None, lse=None, workspace=None, entropy=None):
        """f2: log-probs of the packed actions straight from the final hidden states and the LM-head weight
        (echo_lmhead_logp: the [tokens x vocab] logits are never materialised), e.g. to recompute old_logp or the
        reference model's ref_logp.  hidden: bf16 [n x d] rows aligned with the packed tokens [0, n)."""
        n, d = hidden.shape
        out = torch.empty(n, dtype=torch.float32, device=self.device) if out is None else out
        if workspace is None:
            workspace = torch.empty(abi.echo_lmhead_workspace_bytes(n, self.V) // 4 + 1, dtype=torch.float32,
                                    device=self.device)
        abi.echo_lmhead_logp(hidden, weight, n, d, self.V, self.tok_action[:n], out, lse, workspace,
                             tok_entropy=entropy)
        self.launches += abi.LAUNCHES["echo_lmhead_logp"]
        return out

    def loss_from_hidden(self, hidden, weight, row0: int, dhidden, dweight, *, accumulate=True, clip_low=0.2,
                         clip_high=0.2, kl_coef=0.0, grad_scale=1.0, tok_adv=None, tok_weight=None, clip_dual=0.0,
                         kl_estimator=abi.ECHO_KL_K3, entropy_coef=0.0, chunk_rows=8192, scratch=None,
                         mode="chunked", tok_entropy=None):
        """f2 training step through the LM head for packed rows [row0, row0 + n): dhidden = dL/dh into ``dhidden``
        (f32 [n x d]) and dL/dW added to (``accumulate``) or written over ``dweight`` (f32 [V x d]); per-token outputs
        land in tok_logp / tok_loss / tok_flags as with ``loss``.  No [n x V] logits buffer: at most a
        [chunk_rows x V] bf16 one.  ``scratch``: optional dict of reusable device buffers (keyed by name).

        mode "chunked" (default, echo_lmhead_policy_loss_fwd_bwd): per chunk, z = h W^T stored as bf16 by the tcgen05
            GEMM, the fused (3)-(5) kernel in place, dhidden / dweight on libecho's tcgen05 GEMM (6 d V flops per
            token).
        mode "recompute": (3) echo_lmhead_logp (logp, lse, entropy without the logits), (4) echo_loss_from_logp,
            (5) + backward echo_lmhead_backward with D recomputed from h and W on the tensor cores (8 d V flops per
            token; logits never rounded to bf16)."""
        n, d = hidden.shape
        sl = slice(row0, row0 + n)
        sc = {} if scratch is None else scratch
        dev = self.device
        if mode == "chunked":
            chunk = max(1, min(chunk_rows, n))
            cfg = abi.LossConfig(clip_low, clip_high, clip_dual, kl_coef, grad_scale, kl_estimator, entropy_coef)
            ws = sc.get("zc")
            numel = chunk * abi.echo_lmhead_dlogits_ld(self.V)
            if ws is None or ws.numel() < numel:
                ws = sc["zc"] = torch.empty(numel, dtype=torch.bfloat16, device=dev)
            ref = self.tok_ref[sl] if (self.tok_ref is not None and kl_coef > 0) else None
            abi.echo_lmhead_policy_loss_fwd_bwd(
                hidden, weight, n, d, self.V, self.tok_action[sl], self.tok_old[sl], ref, self.tok_slot[sl],
                self.adv_slot, None if tok_adv is None else tok_adv[sl], None if tok_weight is None else tok_weight[sl],
                self.stats1[0:1], cfg, self.tok_logp[sl], self.tok_loss[sl], self.tok_flags[sl],
                None if tok_entropy is None else tok_entropy[sl], dhidden, dweight, accumulate, ws, chunk)
            if n > 0:
                self.launches += abi.LMHEAD_LOSS_LAUNCHES_PER_CHUNK * ((n + chunk - 1) // chunk)
            return
        if mode != "recompute":
            raise ValueError(f"loss_from_hidden: unknown mode {mode!r}")

        def buf(name, numel, dtype):
            t = sc.get(name)
            if t is None or t.numel() < numel or t.dtype != dtype:
                t = torch.empty(max(numel, 1), dtype=dtype, device=dev)
                sc[name] = t
            return t[:numel]

        ent_on = entropy_coef > 0
        lse = buf("lse", n, torch.float32)
        ent = buf("entropy", n, torch.float32) if ent_on else None
        coef = buf("coef", n, torch.float32)
        ecoef = buf("ecoef", n, torch.float32) if ent_on else None
        ws = buf("ws", abi.echo_lmhead_workspace_bytes(n, self.V) // 4 + 1, torch.float32)
        abi.echo_lmhead_logp(hidden, weight, n, d, self.V, self.tok_action[sl], self.tok_logp[sl], lse, ws,
                             tok_entropy=ent)
        cfg = abi.LossConfig(clip_low, clip_high, clip_dual, kl_coef, grad_scale, kl_estimator, entropy_coef)
        ref = self.tok_ref[sl] if (self.tok_ref is not None and kl_coef > 0) else None
        abi.echo_loss_from_logp(n, self.tok_logp[sl], ent, self.tok_old[sl], ref, self.tok_slot[sl], self.adv_slot,
                                None if tok_adv is None else tok_adv[sl], None if tok_weight is None else tok_weight[sl],
                                self.stats1[0:1], cfg, self.tok_loss[sl], self.tok_flags[sl], coef, ecoef)
        chunk = max(1, min(chunk_rows, n))
        dz = buf("dz", chunk * abi.echo_lmhead_dlogits_ld(self.V), torch.bfloat16)
        abi.echo_lmhead_backward(hidden, weight, n, d, self.V, self.tok_action[sl], lse, coef, ecoef, ent, dhidden,
                                 dweight, accumulate, dz, chunk)
        if n > 0:
            self.launches += (abi.LAUNCHES["echo_lmhead_logp"] + abi.LAUNCHES["echo_loss_from_logp"] +
                              abi.BACKWARD_LAUNCHES_PER_CHUNK * ((n + chunk - 1) // chunk))

    # ------------------------------------------------------------------ (3)-(5)
    def loss(self, logits: torch.Tensor, row0: int, *, clip_low=0.2, clip_high=0.2, kl_coef=0.0, grad_scale=1.0,
             algo=None, stream=None, tok_adv=None, tok_weight=None, clip_dual=0.0, kl_estimator=abi.ECHO_KL_K3,
             entropy_coef=0.0, tok_entropy=None):
        """Fused loss fwd+bwd over packed rows [row0, row0 + logits.shape[0]); logits become dlogits.

        f4 options (echo_policy_loss_fwd_bwd_v2): ``tok_adv`` / ``tok_weight`` are full-length per-token device
        arrays (per-token advantages, e.g. GAE; per-token loss weights, e.g. sequence-mean), ``clip_dual`` and
        ``kl_estimator`` select the dual clip and the KL estimator, ``entropy_coef`` the entropy bonus; ``tok_entropy``
        (full-length f32 device array, nullable) receives the per-token entropies."""
        n_rows, ld = logits.shape
        sl = slice(row0, row0 + n_rows)
        ref = self.tok_ref[sl] if (self.tok_ref is not None and kl_coef > 0) else None
        if (tok_adv is None and tok_weight is None and clip_dual == 0.0 and kl_estimator == abi.ECHO_KL_K3
                and entropy_coef == 0.0 and tok_entropy is None):
            abi.echo_policy_loss_fwd_bwd(logits, self.edtype, n_rows, self.V, ld, self.tok_action[sl], self.tok_old[sl],
                                         ref, self.tok_slot[sl], self.adv_slot, self.stats1[0:1], clip_low, clip_high,
                                         kl_coef, grad_scale, self.tok_logp[sl], self.tok_loss[sl], self.tok_flags[sl],
                                         stream=stream, algo=algo)
        else:
            cfg = abi.LossConfig(clip_low, clip_high, clip_dual, kl_coef, grad_scale, kl_estimator, entropy_coef)
            abi.echo_policy_loss_fwd_bwd_v2(logits, self.edtype, n_rows, self.V, ld, self.tok_action[sl],
                                            self.tok_old[sl], ref, self.tok_slot[sl], self.adv_slot,
                                            None if tok_adv is None else tok_adv[sl],
                                            None if tok_weight is None else tok_weight[sl], self.stats1[0:1], cfg,
                                            self.tok_logp[sl], self.tok_loss[sl], self.tok_flags[sl],
                                            tok_entropy=None if tok_entropy is None else tok_entropy[sl],
                                            algo=abi.ECHO_ALGO_AUTO if algo is None else algo, stream=stream)
        self.launches += abi.LAUNCHES["echo_policy_loss_fwd_bwd"] if n_rows > 0 else 0

    # ------------------------------------------------------------------ statistics
    def finish(self, read_back: bool = True, tok_weight=None) -> dict | None:
        n = self.pack_info.n_tokens
        abi.echo_loss_stats(n, self.tok_loss, self.tok_logp, self.tok_old,
                            self.tok_ref if self.tok_ref is not None else None, self.tok_flags, self.ws,
                            self.loss_stats, tok_weight=tok_weight)
        self.launches += abi.LAUNCHES["echo_loss_stats"]
        reduce_loss_stats_(self.loss_stats, self.group)
        if not read_back:
            return None
        self.stats_host[: len(STATS1)].copy_(self.stats1, non_blocking=True)
        self.stats_host[len(STATS1):].copy_(self.loss_stats, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        v = self.stats_host.tolist()
        out = dict(zip(STATS1, v[: len(STATS1)]))
        out.update({"loss/" + k: x for k, x in zip(LOSS_STATS, v[len(STATS1):])})
        if tok_weight is not None:
            out["loss"] = out["loss/sum_weighted_loss"]
        else:
            out["loss"] = out["loss/sum_loss"] / out["n_tokens"] if out["n_tokens"] else 0.0
        return out

    def d2h_bytes(self) -> int:
        return abi.PACK_RESULT_BYTES + self.stats_host.numel() * 8

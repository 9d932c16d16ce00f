"""Expert parallelism for the MoQE layer: experts sharded across ranks, token
rows dispatched to the expert owners and returned with an all-to-all.

The reference is single-process (SPEC.md:330 lists distributed expert
parallelism as a non-goal); this is the B200 scale-out of the same layer math
(BASELINE config 4: 128 experts, top-2, experts sharded 128/G over G GPUs).
Rank g owns experts [g*E/G, (g+1)*E/G) and holds its own tokens; the router
weights are replicated.

One forward:
  1. route local tokens (exact fp32 router kernel; global expert ids + gates)
  2. group (token, slot) rows by owner rank, ascending token order (stable); on the GPU
     one kernel pair does it (k_ep_plan + k_ep_pack, csrc/ep.cu: moqe_gpu_ep_dispatch)
  3. exchange per-rank counts (one small all_to_all + one read of G counts), then ONE
     all_to_all of packed records: the fp16 row with the owner-local expert id and the
     gate bit-cast into 4 trailing fp16 slots (NCCL over NVLink on GPU, gloo on CPU)
  4. owners run the expert FFN on the received rows (moqe_gpu_expert_ffn: the
     same decode / tcgen05 kernels as moe_forward; out = gate * FFN(row))
  5. all_to_all the gate-weighted rows back, fp16 by default (half the return bytes;
     return_dtype=torch.float32 keeps the bit-exact fp32 return)
  6. combine: out[t] = sum over t's slots, added onto zero (two addends,
     commutative -> deterministic); on the GPU k_ep_combine (moqe_gpu_ep_combine).
The CPU form of steps 2 and 6 (torch.sort / bincount / index_add_) only serves the gloo
tests of the exchange logic; CUDA tensors always take the kernels.
With an fp32 return the output equals the single-GPU moe_forward of the whole layer bit for
bit (combine order identical for top-1/top-2); the fp16 return rounds each gated row once.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist


def shard_range(n_experts: int, world: int, rank: int) -> Tuple[int, int]:
    if n_experts % world:
        raise ValueError(f"{n_experts} experts do not shard evenly over {world} ranks")
    per = n_experts // world
    return rank * per, (rank + 1) * per


def dispatch_plan(expert: torch.Tensor, n_experts: int, world: int):
    """Flatten (token, slot) assignments and order them by owner rank
    (stable: ascending token order inside each destination).

    Returns (order, tok, dest_sorted, send_counts): `order` indexes the flat
    assignment list, tok[i] is the source token of flat assignment i."""
    T = expert.shape[0]
    k = 1 if expert.dim() == 1 else expert.shape[1]
    flat = expert.reshape(-1).long()
    tok = torch.arange(T, device=expert.device).repeat_interleave(k)
    per = n_experts // world
    dest = flat // per
    dest_sorted, order = torch.sort(dest, stable=True)
    send_counts = torch.bincount(dest, minlength=world)
    return order, tok, dest_sorted, send_counts


class ExpertParallelMoE:
    """A sharded MoE FFN layer: this rank's ExpertBank + replicated router.

    `route_fn(h) -> (expert [T,k] int32 global ids, gate [T,k] f32)` and
    `expert_fn(x, local_expert, gate) -> gate-weighted rows` default to the
    GPU kernels; tests inject CPU stand-ins to check the exchange logic."""

    def __init__(self, bank, router: torch.Tensor, n_experts: int, top_k: int = 2,
                 group: Optional[dist.ProcessGroup] = None,
                 route_fn: Optional[Callable] = None, expert_fn: Optional[Callable] = None,
                 path: str = "auto", return_dtype: torch.dtype = torch.float16):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.E = n_experts
        self.lo, self.hi = shard_range(n_experts, self.world, self.rank)
        self.top_k = top_k
        self.bank = bank
        self.router = router
        self.path = path
        self.return_dtype = return_dtype
        if route_fn is None or expert_fn is None:
            from . import api
        self.route_fn = route_fn or (lambda h: api.route(h, self.router, self.top_k))
        # ids come from this layer's own router: no host-side range check (no sync)
        self.expert_fn = expert_fn or (lambda x, e, g: api.expert_ffn(x, self.bank, e, g, path=self.path,
                                                                         out_dtype=self.return_dtype,
                                                                         validate=False))

    def _forward_device(self, h: torch.Tensor, ex: torch.Tensor, gate: torch.Tensor) -> torch.Tensor:
        """The GPU step: dispatch and combine in this package's kernels (ep.cu), one host
        read (the G send / receive counts + the id-range flag, one copy)."""
        from . import api
        T, d = h.shape
        k = ex.shape[1]
        rec, pos, send_counts, err = api.ep_dispatch(h, ex, gate, self.E, self.world)
        recv_counts = torch.empty_like(send_counts)
        self._a2a(recv_counts, send_counts, None, None)
        host = torch.cat([send_counts, recv_counts, err.to(torch.int64)]).tolist()
        G = self.world
        s_split, r_split = host[:G], host[G:2 * G]
        if host[2 * G]:
            raise IndexError("ep: expert id out of range")
        R = int(sum(r_split))
        recv = torch.empty((R, d + 4), dtype=torch.float16, device=h.device)
        self._a2a(recv, rec, r_split, s_split)
        rmeta = recv[:, d:].view(torch.int32)
        y = self.expert_fn(recv[:, :d], rmeta[:, 0].contiguous(),
                           rmeta[:, 1].contiguous().view(torch.float32)).to(self.return_dtype).contiguous()
        back = torch.empty((T * k, d), dtype=self.return_dtype, device=h.device)
        self._a2a(back, y, s_split, r_split)
        return api.ep_combine(back, pos, T, k)

    def _a2a(self, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits) -> None:
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def forward(self, h: torch.Tensor) -> torch.Tensor:
        T, d = h.shape
        ex, gate = self.route_fn(h)
        ex = ex.reshape(T, -1)
        gate = gate.reshape(T, -1)
        if h.is_cuda:
            return self._forward_device(h, ex, gate)
        order, tok, dest_sorted, send_counts = dispatch_plan(ex, self.E, self.world)
        src_tok = tok[order]
        R_send = src_tok.shape[0]
        # packed records: [row (d fp16) | expert id (i32) | gate (f32)] as d + 4 fp16 slots
        rec = torch.empty((R_send, d + 4), dtype=torch.float16, device=h.device)
        rec[:, :d] = h.index_select(0, src_tok)
        meta = rec[:, d:].view(torch.int32)  # two int32 words per record
        meta[:, 0] = (ex.reshape(-1)[order] - dest_sorted * (self.E // self.world)).to(torch.int32)
        meta[:, 1] = gate.reshape(-1)[order].to(torch.float32).view(torch.int32)

        # 1) counts (the only host read: G integers, the all_to_all split sizes)
        recv_counts = torch.empty_like(send_counts)
        self._a2a(recv_counts, send_counts, None, None)
        s_split = send_counts.tolist()
        r_split = recv_counts.tolist()
        R = int(sum(r_split))
        # 2) packed rows + metadata to the owners, one collective
        recv = torch.empty((R, d + 4), dtype=torch.float16, device=h.device)
        self._a2a(recv, rec, r_split, s_split)
        rmeta = recv[:, d:].view(torch.int32)
        recv_exp = rmeta[:, 0].contiguous()
        recv_gate = rmeta[:, 1].contiguous().view(torch.float32)
        # 3) owner-side expert FFN (gate-weighted rows)
        y = self.expert_fn(recv[:, :d], recv_exp, recv_gate).to(self.return_dtype).contiguous()
        # 4) back to the sources, in the order they were sent
        back = torch.empty((R_send, d), dtype=self.return_dtype, device=h.device)
        self._a2a(back, y, s_split, r_split)
        # 5) combine the top-k slots (<= 2 addends onto zero: order-independent)
        out = torch.zeros((T, d), dtype=torch.float32, device=h.device)
        out.index_add_(0, src_tok, back.to(torch.float32))
        return out

"""Thin torch-tensor wrappers over the C-ABI kernels (no logic, no fallback)."""

from __future__ import annotations

import torch

from . import _native as N

C128 = torch.complex128


def _c128(t: torch.Tensor, name: str):
    if t.dtype != C128:
        raise TypeError(f"{name} must be complex128, got {t.dtype}")
    N.require_cuda(t)


def _span(t: torch.Tensor):
    """[first, last] byte addresses touched by a (possibly strided) tensor."""
    if t.numel() == 0:
        return (0, -1)
    last = sum((n - 1) * st for n, st in zip(t.shape, t.stride()))
    return (t.data_ptr(), t.data_ptr() + (last + 1) * t.element_size() - 1)


def _no_alias(a: torch.Tensor, b: torch.Tensor):
    """Every output row depends on all input rows and CTAs write as they go, so in == out (or
    overlapping views) would be a read-after-write race across CTAs.  Column blocks of one
    buffer interleave without sharing bytes: those are compared exactly."""
    (a0, a1), (b0, b1) = _span(a), _span(b)
    if a1 < b0 or b1 < a0:
        return
    if a.stride() == b.stride() and a.shape == b.shape and a.stride(-2) >= a.shape[-1]:
        off = abs(a0 - b0) // a.element_size() % a.stride(-2)
        if off >= a.shape[-1] and a.stride(-2) - off >= a.shape[-1]:
            return   # disjoint column blocks of the same row-major buffer
    raise ValueError("transform: input and output overlap (in-place transforms are not supported)")


def time_transform(T: torch.Tensor, v: torch.Tensor, out: torch.Tensor | None = None,
                   stream=None) -> torch.Tensor:
    """out[..., l, :] = sum_k T[l, k] v[..., k, :] on the DMMA kernel (K3).

    v: (n_t, N) or (B, n_t, N) complex128 with unit column stride (rows may be
    strided).  Returns a new tensor (or writes `out`)."""
    _c128(T, "T")
    _c128(v, "v")
    nt = T.shape[0]
    if T.shape != (nt, nt) or v.shape[-2] != nt:
        raise N.DimensionMismatch(N.ERR_DIM, f"transform: T {tuple(T.shape)} vs v {tuple(v.shape)}")
    T = T.contiguous()
    squeeze = v.dim() == 2
    vb = v.unsqueeze(0) if squeeze else v
    if vb.stride(-1) != 1:
        vb = vb.contiguous()
    if out is None:
        out = torch.empty(v.shape, dtype=C128, device=v.device)
    ob = out.unsqueeze(0) if out.dim() == 2 else out
    if ob.stride(-1) != 1 or ob.shape != vb.shape:
        raise N.DimensionMismatch(N.ERR_DIM, "transform: bad output tensor")
    B, _, ncols = vb.shape
    _no_alias(vb, ob)
    N.check(N.lib().stfem_time_transform(
        N.ptr(T), nt, N.ptr(vb), vb.stride(-2), N.ptr(ob), ob.stride(-2), ncols, B,
        vb.stride(0) if B > 1 else 0, ob.stride(0) if B > 1 else 0, N.stream_ptr(stream)))
    return out


def transform_pair_fwd(pairs, v: torch.Tensor, out: torch.Tensor | None = None, stream=None,
                       out_cols: torch.Tensor | None = None) -> torch.Tensor:
    """G = Y v through the eigenpair-paired kernel (K3p forward); `pairs` is a
    paired_transform.DevicePairs.  Same shapes/strides contract as time_transform.
    out_cols (int32, one per column of v): column j of the result goes to column
    out_cols[j] of `out`, which may then be wider than v (a column block of v scattered
    into the whole stack)."""
    _c128(v, "v")
    nt = pairs.nt
    if v.shape[-2] != nt:
        raise N.DimensionMismatch(N.ERR_DIM, f"transform: n_t {nt} vs v {tuple(v.shape)}")
    vb = v.unsqueeze(0) if v.dim() == 2 else v
    if vb.stride(-1) != 1:
        vb = vb.contiguous()
    if out is None:
        out = torch.empty(v.shape, dtype=C128, device=v.device)
    ob = out.unsqueeze(0) if out.dim() == 2 else out
    if ob.stride(-1) != 1 or ob.shape[:-1] != vb.shape[:-1] or (out_cols is None and ob.shape != vb.shape):
        raise N.DimensionMismatch(N.ERR_DIM, "transform: bad output tensor")
    B, _, ncols = vb.shape
    _no_alias(vb, ob)
    if out_cols is not None and (out_cols.dtype != torch.int32 or out_cols.numel() != ncols or not out_cols.is_cuda):
        raise N.DimensionMismatch(N.ERR_DIM, "transform: out_cols must be int32 on the device, one per column")
    N.check(N.lib().stfem_transform_pair_fwd_map(
        N.ptr(pairs.A_fwd), pairs.mrows_fwd, nt, N.ptr(pairs.rows_fwd), N.ptr(pairs.scale_fwd),
        pairs.rows_fwd.shape[0], N.ptr(vb), vb.stride(-2), N.ptr(ob), ob.stride(-2), ncols, B,
        vb.stride(0) if B > 1 else 0, ob.stride(0) if B > 1 else 0,
        N.ptr(out_cols) if out_cols is not None else None, N.stream_ptr(stream)))
    return out


def pair_mix(pairs, w: torch.Tensor, stream=None) -> torch.Tensor:
    """In-place pre-pass of the paired back transform over every column of w (needed once before
    transform_pair_back(..., in_cols=..., mixed=True) calls on column blocks)."""
    _c128(w, "w")
    wb = w.unsqueeze(0) if w.dim() == 2 else w
    if wb.stride(-1) != 1 or wb.shape[-2] != pairs.nt:
        raise N.DimensionMismatch(N.ERR_DIM, "pair_mix: w needs n_t rows and unit column stride")
    B, _, ncols = wb.shape
    N.check(N.lib().stfem_pair_mix(N.ptr(pairs.mix_rows), N.ptr(pairs.mix_coef), pairs.mix_rows.shape[0], N.ptr(wb),
                                   wb.stride(-2), ncols, B, wb.stride(0) if B > 1 else 0, N.stream_ptr(stream)))
    return w


def transform_pair_back(pairs, w: torch.Tensor, out: torch.Tensor | None = None, stream=None,
                        in_cols: torch.Tensor | None = None, mixed: bool = False) -> torch.Tensor:
    """Psi = X w through the paired kernel (K3p back).  `w` is CLOBBERED (the
    in-place pair pre-pass); it must have unit column stride.
    in_cols (int32, one per column of out): result column j reads column in_cols[j] of w (w may
    then be wider than out); the pre-pass must already have run over all of w (`pair_mix`,
    mixed=True)."""
    _c128(w, "w")
    nt = pairs.nt
    if w.shape[-2] != nt:
        raise N.DimensionMismatch(N.ERR_DIM, f"transform: n_t {nt} vs w {tuple(w.shape)}")
    wb = w.unsqueeze(0) if w.dim() == 2 else w
    if wb.stride(-1) != 1:
        raise N.DimensionMismatch(N.ERR_DIM, "transform_pair_back: w needs unit column stride (updated in place)")
    if out is None:
        out = torch.empty(w.shape, dtype=C128, device=w.device)
    ob = out.unsqueeze(0) if out.dim() == 2 else out
    if ob.stride(-1) != 1 or ob.shape[:-1] != wb.shape[:-1] or (in_cols is None and ob.shape != wb.shape):
        raise N.DimensionMismatch(N.ERR_DIM, "transform: bad output tensor")
    B, _, ncols = ob.shape
    _no_alias(wb, ob)
    if in_cols is not None:
        if in_cols.dtype != torch.int32 or in_cols.numel() != ncols or not in_cols.is_cuda or not mixed:
            raise N.DimensionMismatch(N.ERR_DIM, "transform: in_cols must be int32 on the device, one per output "
                                                 "column, after pair_mix over all of w (mixed=True)")
    N.check(N.lib().stfem_transform_pair_back_map(
        N.ptr(pairs.A_back), nt, N.ptr(pairs.mix_rows), N.ptr(pairs.mix_coef),
        0 if mixed else pairs.mix_rows.shape[0],
        N.ptr(wb), wb.stride(-2), N.ptr(ob), ob.stride(-2), ncols, B,
        wb.stride(0) if B > 1 else 0, ob.stride(0) if B > 1 else 0,
        N.ptr(in_cols) if in_cols is not None else None, N.stream_ptr(stream)))
    return out

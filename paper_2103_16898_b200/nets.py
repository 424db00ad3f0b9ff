"""CNNs of the paper's GPU-offloaded training step, built on the sm_100a kernels.

The reference contains no CNN (its trainer is a logistic toy, workload.py:48-71); the
models follow the paper's prose and BASELINE.json's configs (defined in DESIGN.md):
  SmallCNN     PAPER.md:441-443 "4 conv + BN, 2 FC, Adam lr 1e-3" on 32x32x3, 10 classes
  ResNet18     CIFAR variant (3x3 stem, no max-pool), BASELINE.json configs[2]
  DenseNet121  growth 32, blocks (6,12,24,16), 1-channel 224x224 stem, 2 classes, configs[3]

Execution model: every buffer is allocated once for a fixed per-rank batch (build()), the
step is a fixed launch sequence (forward, loss, backward, fused Adam) on the current
stream, so it can be captured into one CUDA graph and replayed.  Parameters live in one
flat fp32 buffer (plus grads, Adam moments and a bf16 compute copy) -- one Adam launch and
one NCCL bucket space for data parallelism.

Numerics (the contract the CPU restatement oracle/cnn_ref.py follows): conv/FC operands
bf16, fp32 accumulation in TMEM, activations stored bf16, BN statistics and all gradients
of parameters fp32, activation gradients stored bf16, master weights fp32.
"""
from __future__ import annotations

import math
import os

import torch

from . import kernels as K

BF16, F32 = torch.bfloat16, torch.float32
_UNFUSED_HEAD = os.environ.get("CVB_UNFUSED_HEAD", "0") not in ("", "0")
_NO_OVERLAP = os.environ.get("CVB_NO_OVERLAP", "0") not in ("", "0")
# residual BN layers hand their ReLU mask to the backward as bits (A/B: CVB_NO_RELU_MASK=1 re-reads y)
_RELU_MASK = not os.environ.get("CVB_NO_RELU_MASK") and not os.environ.get("CVB_BN_UNFUSED")
# 3x3 stride-2 dgrads as two row-parity convs (A/B: CVB_NO_DGRAD_ROWS=1 keeps the four parity classes)
_DGRAD_ROWS = not os.environ.get("CVB_NO_DGRAD_ROWS")


class _nullctx:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False
ALIGN = 64  # elements; keeps every parameter view 128-byte aligned (TMA needs 16 B)


def _pad16(n):
    return (n + 15) // 16 * 16


class ParamStore:
    """Flat fp32 master / grad / Adam state + bf16 compute copy with per-parameter views."""

    def __init__(self):
        self.specs = []      # (name, shape, init cpu tensor)
        self.logical = 0     # parameter count without layout padding
        self.grad_hook = None   # data parallelism: called with parameter names whose grads are final
        self.side = None        # single GPU: stream the conv weight gradients run on, beside the dgrads
        self.side_used = False

    def grad_ready(self, *names):
        """Backward marks parameters whose gradients are final (launches bucket all-reduces)."""
        if self.grad_hook is not None:
            self.grad_hook(names)

    def add(self, name, init: torch.Tensor, logical: int | None = None):
        self.specs.append((name, tuple(init.shape), init.float()))
        self.logical += init.numel() if logical is None else logical
        return name

    def want_flip(self, name):
        """Keep a flipped/transposed bf16 copy [cin][kh][kw][cout] of conv weight `name` for
        stride-1 dgrad, refreshed for all layers in one launch after every optimiser step."""
        if name not in getattr(self, "flip_names", []):
            self.flip_names = getattr(self, "flip_names", []) + [name]

    def want_class_weights(self, name, pad):
        """Keep the stride-2 dgrad's per-output-parity class weight matrices of conv weight `name`
        (csrc/umma_gemm.cu cvb_conv2d_dgrad_s2 layout), refreshed by the same batched launch."""
        if name not in dict(getattr(self, "class_names", [])):
            self.class_names = getattr(self, "class_names", []) + [(name, pad)]

    def want_row_weights(self, name, pad):
        """Keep the row-parity weight matrices of a 3x3 pad-1 stride-2 conv (cvb_conv2d_dgrad_s2_rows
        layout), refreshed by the same batched launch."""
        if name not in dict(getattr(self, "row_names", [])):
            self.row_names = getattr(self, "row_names", []) + [(name, pad)]

    def flip_all(self):
        if self.flip_n:
            K.transpose_batched(self.pb, self.fb, self.flip_desc, self.flip_n, self.flip_max, self.flip_bytes)

    def finalize(self, device):
        offs, off = {}, 0
        for name, shape, _ in self.specs:
            offs[name] = off
            n = math.prod(shape)
            off += (n + ALIGN - 1) // ALIGN * ALIGN
        self.total = off
        self.p32 = torch.zeros(off, dtype=F32, device=device)
        # one extra aligned slot after the parameters: the step's decrypt verdict (0/1 per rank,
        # summed by the gradient all-reduce like any gradient) that gates the optimiser
        self.g32 = torch.zeros(off + ALIGN, dtype=F32, device=device)
        self.verdict_slot = self.g32[off:off + 1]
        self.m = torch.zeros(off, dtype=F32, device=device)
        self.v = torch.zeros(off, dtype=F32, device=device)
        self.pb = torch.zeros(off, dtype=BF16, device=device)
        self.p, self.g, self.b, self.offsets = {}, {}, {}, offs
        for name, shape, init in self.specs:
            o, n = offs[name], math.prod(shape)
            self.p[name] = self.p32[o:o + n].view(shape)
            self.g[name] = self.g32[o:o + n].view(shape)
            self.b[name] = self.pb[o:o + n].view(shape)
            self.p[name].copy_(init.to(device))
        K.cast_f32_bf16(self.p32, self.pb)
        # flipped dgrad weights: one flat bf16 buffer, one launch for all layers
        shapes = {name: shape for name, shape, _ in self.specs}
        # batched transpose jobs {src, dst, rows, cols, src ld, dst ld}: flipped stride-1 dgrad
        # weights [cin][kh][kw][cout] (one job per tap, tap t -> taps-1-t) and stride-2 parity-class
        # weights [ci][t][co] per class (one job per class tap)
        names = getattr(self, "flip_names", [])
        desc, self.f, self.cw, foff, self.flip_max = [], {}, {}, 0, 1
        for name in names:
            cout, kh, kw, cin = shapes[name]
            n, taps = cout * kh * kw * cin, kh * kw
            for t in range(taps):
                desc += [offs[name] + t * cin, foff + (taps - 1 - t) * cout, cout, cin, taps * cin, taps * cout]
            self.f[name] = (foff, (cin, kh, kw, cout))
            foff += (n + ALIGN - 1) // ALIGN * ALIGN
            self.flip_max = max(self.flip_max, cout * cin)
        for name, pad in getattr(self, "class_names", []):
            cout, kh, kw, cin = shapes[name]
            n, taps, coff = cout * kh * kw * cin, kh * kw, foff
            for _, taplist in K.dgrad_s2_classes(kh, kw, pad):
                nt = len(taplist)
                for t, (y, x) in enumerate(taplist):
                    desc += [offs[name] + (y * kw + x) * cin, coff + t * cout, cout, cin, taps * cin, nt * cout]
                coff += cin * nt * cout
            self.cw[name] = (foff, (n,))
            foff += (n + ALIGN - 1) // ALIGN * ALIGN
            self.flip_max = max(self.flip_max, cout * cin)
        self.rw = {}
        for name, pad in getattr(self, "row_names", []):
            cout, kh, kw, cin = shapes[name]
            desc += K.dgrad_s2_row_jobs(offs[name], kh, kw, cin, cout, pad, foff)
            self.rw[name] = (foff, (12 * cin * cout,))
            foff += (12 * cin * cout + ALIGN - 1) // ALIGN * ALIGN
            self.flip_max = max(self.flip_max, cout * cin)
        self.fb = torch.zeros(max(1, foff), dtype=BF16, device=device)
        for name, (o, shp) in list(self.f.items()):
            self.f[name] = self.fb[o:o + math.prod(shp)].view(shp)
        for name, (o, shp) in list(self.cw.items()):
            self.cw[name] = self.fb[o:o + shp[0]]
        for name, (o, shp) in list(self.rw.items()):
            self.rw[name] = self.fb[o:o + shp[0]]
        self.flip_n = len(desc) // 6
        self.flip_bytes = 4 * foff
        self.flip_desc = torch.tensor(desc if desc else [0], dtype=torch.int64, device=device)
        self.flip_all()
        self.step_dev = torch.zeros(1, dtype=torch.int32, device=device)
        self.sched = torch.zeros(4, dtype=F32, device=device)   # bias-correction factors + Adam's CTA counter

    def state_cpu(self):
        return {name: self.p[name].detach().cpu().clone() for name, _, _ in self.specs}


def _uniform(gen, shape, bound):
    return (torch.rand(shape, generator=gen) * 2 - 1) * bound


class Scratch:
    """Shared scratch for split-K partials, BN partials and flipped weights."""

    def __init__(self):
        self.part_floats = 1
        self.bn_floats = 1
        self.flip_elems = 1
        self.up_elems = 1

    def finalize(self, device):
        self.part = torch.empty(self.part_floats, dtype=F32, device=device)
        self.bnws = torch.empty(self.bn_floats, dtype=F32, device=device)
        self.flip = torch.empty(self.flip_elems, dtype=BF16, device=device)
        self.up = torch.empty(self.up_elems, dtype=BF16, device=device)


MAX_SPLITS = 148
PART_CAP = 16 << 20   # floats of split-K partial workspace (64 MB)


class ConvBN:
    """conv (no bias) -> batch norm -> [+ residual] -> [ReLU]; NHWC bf16."""

    def __init__(self, ps: ParamStore, name, cin, cout, k, stride, pad, gen, relu=True, cin_real=None,
                 need_dgrad=True):
        self.name, self.cin, self.cout, self.k, self.s, self.pad = name, cin, cout, k, stride, pad
        self.relu, self.need_dgrad = relu, need_dgrad
        cin_real = cin if cin_real is None else cin_real
        self.cin_real = cin_real
        # DenseNet's 7x7 stride-2 stem on 8-channel (1 real) input: computed as a 4x4 stride-1
        # conv on the 2x2 space-to-depth input (32 channels) -> the halo conv path instead of
        # 49 gathered 16-byte-row boxes per K-block (same result, exact same products)
        self.s2d = (k == 7 and stride == 2 and pad == 3 and cin == 8 and not need_dgrad
                    and not os.environ.get("CVB_NO_S2D"))
        bound = 1.0 / math.sqrt(cin_real * k * k)  # torch default (kaiming_uniform a=sqrt(5))
        w = _uniform(gen, (cout, k, k, cin_real), bound)
        if cin_real != cin:
            w = torch.cat([w, torch.zeros(cout, k, k, cin - cin_real)], dim=3)
        self.W = ps.add(f"{name}.w", w, logical=cout * k * k * cin_real)
        if need_dgrad and stride == 1:
            ps.want_flip(self.W)
        elif need_dgrad and stride == 2:
            ps.want_class_weights(self.W, pad)
            if k == 3 and pad == 1 and _DGRAD_ROWS:
                ps.want_row_weights(self.W, pad)
        self.G = ps.add(f"{name}.gamma", torch.ones(cout))
        self.B = ps.add(f"{name}.beta", torch.zeros(cout))

    def build(self, n, h, w, scratch: Scratch, device):
        self.n, self.h, self.w = n, h, w
        self.oh, self.ow = K.conv_out_hw(h, w, self.k, self.s, self.pad)
        self.rows = n * self.oh * self.ow
        if self.s2d:
            self.xs = torch.empty(n, h // 2, w // 2, 4 * self.cin, dtype=BF16, device=device)
            self.ws = torch.empty(self.cout, 4, 4, 4 * self.cin, dtype=BF16, device=device)
            self.dws = torch.empty(self.cout, 16 * 4 * self.cin, dtype=F32, device=device)
        self.flops = 2 * self.rows * self.cout * self.k * self.k * self.cin_real   # algorithmic, per pass
        self.z = torch.empty(n, self.oh, self.ow, self.cout, dtype=BF16, device=device)
        self.dz = torch.empty_like(self.z)
        self.mean = torch.zeros(self.cout, dtype=F32, device=device)
        self.rstd = torch.zeros(self.cout, dtype=F32, device=device)
        self.run_mean = torch.zeros(self.cout, dtype=F32, device=device)
        self.run_var = torch.ones(self.cout, dtype=F32, device=device)
        # residual layers keep y's ReLU mask as bits (rows x cout/8 bytes) for the backward instead
        # of re-reading y (1/16 of the bytes); allocated on the first residual forward
        self.mask = None
        self.wcount = self.cout * self.k * self.k * self.cin
        scratch.part_floats = max(scratch.part_floats, min(MAX_SPLITS * self.wcount, max(PART_CAP, 8 * self.wcount)))
        scratch.bn_floats = max(scratch.bn_floats, K._lib_bound().cvb_bn_workspace_floats(self.rows, self.cout))
        if self.need_dgrad:
            scratch.flip_elems = max(scratch.flip_elems, self.cout * self.k * self.k * self.cin)
            if self.s == 2:
                scratch.up_elems = max(scratch.up_elems, n * (2 * self.oh - 1) * (2 * self.ow - 1) * self.cout)
        self.scratch = scratch
        return self.oh, self.ow

    def forward(self, ps: ParamStore, x, out, res=None, out_coff=0, cin=None):
        """x: [n,h,w,cs] (channels [0,cin)); out: [n,oh,ow,ocs] written at channel out_coff."""
        if self.s2d:
            K.space_to_depth2(x, self.xs)
            K.s2d_weights(ps.b[self.W], self.ws)
            K.conv2d_fwd(self.xs, self.ws, 1, 2, out=self.z, out_hw=(self.oh, self.ow), acct_flops=self.flops)
        else:
            K.conv2d_fwd(x, ps.b[self.W], self.s, self.pad, out=self.z, cin=cin if cin is not None else self.cin,
                         acct_flops=self.flops)
        if res is not None and self.relu and self.mask is None and _RELU_MASK:
            self.mask = torch.empty(self.rows, self.cout // 8, dtype=torch.uint8, device=self.z.device)
        K.bn_forward(self.z, self.rows, self.cout, self.cout, self.scratch.bnws, self.mean, self.rstd, ps.p[self.G],
                     ps.p[self.B], out, out.shape[-1], out_coff, relu=self.relu, res=res,
                     rcs=res.shape[-1] if res is not None else 0, run_mean=self.run_mean, run_var=self.run_var,
                     mask=self.mask if res is not None else None)

    def backward(self, ps: ParamStore, dout, x, dx=None, y=None, dres=None, dx_accumulate=False, cin=None,
                 dout_coff=0):
        """dout: grad of this layer's output; y: the output (ReLU mask when a residual was added);
        dres: receives the residual branch's gradient (masked dout); dx: grad wrt x (bf16)."""
        cin = self.cin if cin is None else cin
        dcs = dout.shape[-1]
        dsrc = dout if dout_coff == 0 else dout[..., dout_coff:]
        K.bn_backward(dsrc, dcs, self.z, self.cout, self.rows, self.cout, self.mean, self.rstd, ps.p[self.G],
                      ps.p[self.B], self.scratch.bnws, ps.g[self.G], ps.g[self.B], relu=self.relu,
                      y=y if self.mask is None else None, ycs=y.shape[-1] if y is not None else 0, dx=self.dz,
                      dxcs=self.cout, dz_out=dres, mask=self.mask if y is not None else None)
        if self.s2d:   # wgrad of the 4x4 s2d conv, mapped back onto the 7x7 weights
            count = self.cout * 16 * 4 * self.cin
            maxs = max(1, min(MAX_SPLITS, self.scratch.part.numel() // count))
            part, used = K.conv2d_wgrad_partials(self.dz, self.xs, 4, 4, 1, 2,
                                                 part=self.scratch.part[:maxs * count].view(maxs, self.cout,
                                                                                            16 * 4 * self.cin),
                                                 acct_flops=self.flops)
            K.reduce_splits(part, used, count, self.dws)
            K.s2d_weights_grad(self.dws, ps.g[self.W])
            ps.grad_ready(self.W, self.G, self.B)
            return
        count = self.cout * self.k * self.k * cin
        maxs = max(1, min(MAX_SPLITS, self.scratch.part.numel() // count))
        # single GPU: the weight gradient (split-K wgrad + reduction) runs on the side stream while
        # the dgrad and the next layer's BN backward proceed (both only need dz); the side stream
        # serialises the wgrads, so the shared split-K scratch is never used by two at once
        side = ps.side if dx is not None else None
        if side is not None:
            side.wait_stream(torch.cuda.current_stream())
            ps.side_used = True
        with torch.cuda.stream(side) if side is not None else _nullctx():
            part, used = K.conv2d_wgrad_partials(self.dz, x, self.k, self.k, self.s, self.pad, cin=cin,
                                                 part=self.scratch.part[:maxs * count].view(maxs, self.cout,
                                                                                            self.k * self.k * cin),
                                                 acct_flops=self.flops)
            K.reduce_splits(part, used, count, ps.g[self.W])
            ps.grad_ready(self.W, self.G, self.B)
        if dx is not None:
            wt = self.scratch.flip[:self.cout * self.k * self.k * cin].view(cin, self.k, self.k, self.cout)
            if self.s == 2 and cin == self.cin and self.W in getattr(ps, "rw", {}):
                if K.conv2d_dgrad_s2_rows(self.dz, ps.rw[self.W], cin, dx, accumulate=dx_accumulate,
                                          acct_flops=self.flops):
                    return
            if self.s == 2 and cin == self.cin:
                ready = self.W in ps.cw   # class weights refreshed by ParamStore.flip_all
                if K.conv2d_dgrad_s2(self.dz, ps.b[self.W], self.pad, dx, accumulate=dx_accumulate,
                                     wscratch=ps.cw[self.W] if ready else wt, acct_flops=self.flops,
                                     class_weights_ready=ready):
                    return
            if self.s == 1 and cin == self.cin and self.W in ps.f:
                wt = ps.f[self.W]          # refreshed for every layer by ParamStore.flip_all
            else:
                K.weight_flip(ps.b[self.W], wt)
            src = self.dz
            if self.s == 2:
                uh, uw = 2 * self.oh - 1, 2 * self.ow - 1
                src = self.scratch.up[:self.n * uh * uw * self.cout].view(self.n, uh, uw, self.cout)
                K.zero_upsample(self.dz, src)
            K.conv2d_fwd(src, wt, 1, self.k - 1 - self.pad, out=dx, out_hw=(self.h, self.w),
                         accumulate=dx_accumulate, acct_flops=self.flops)


class Linear:
    """y = x W^T + b with W [out_pad][in] (out padded to 16 so every TMA row stride is legal)."""

    def __init__(self, ps: ParamStore, name, fin, fout, gen):
        self.fin, self.fout, self.fpad = fin, fout, _pad16(fout)
        bound = 1.0 / math.sqrt(fin)
        w = torch.zeros(self.fpad, fin)
        w[:fout] = _uniform(gen, (fout, fin), bound)
        b = torch.zeros(self.fpad)
        b[:fout] = _uniform(gen, (fout,), bound)
        self.W = ps.add(f"{name}.w", w, logical=fout * fin)
        self.Bn = ps.add(f"{name}.b", b, logical=fout)

    @staticmethod
    def _splits(M, N, Kd, bn_cap=256):
        """split-K factor so that the (m, n, split) work units cover the 148 SMs; short K
        (<= 8 K-blocks) and tiny outputs skip split-K -- the partial-sum reduction launch
        would cost more than the GEMM."""
        if Kd <= 512 or M * N <= 64 * 1024:
            return 1
        tiles = -(-M // 128) * -(-N // min(bn_cap, _pad16(N)))
        return max(1, min(-(-Kd // 64), 148 // max(1, tiles)))

    def build(self, batch, scratch):
        B = batch
        # forward: narrow (64-column) N tiles -> 4x more output tiles, 4x fewer split-K partials
        self.bn_fwd = 64 if self.fpad > 64 else 256
        self.s_fwd = self._splits(B, self.fpad, self.fin, bn_cap=self.bn_fwd)
        self.s_wg = self._splits(self.fpad, self.fin, B)
        need = max(self.s_fwd * B * self.fpad, self.s_wg * self.fpad * self.fin if self.s_wg > 1 else 0)
        scratch.part_floats = max(scratch.part_floats, need)
        self.scratch = scratch

    def forward(self, ps, x, out, out_f32=False, relu=False):
        B = x.shape[0]
        fl = 2 * B * self.fout * self.fin
        if self.s_fwd > 1:
            part = self.scratch.part[:self.s_fwd * B * self.fpad].view(self.s_fwd, B, self.fpad)
            K.gemm(x, ps.b[self.W], B, self.fpad, self.fin, 0, 0, out=part, splits=self.s_fwd, acct_flops=fl,
                   max_bn=self.bn_fwd)
            used = K.splits_used(self.fin, self.s_fwd)
            K.reduce_splits_act(part, used, B, self.fpad, out, bias=ps.p[self.Bn], relu=relu)
        else:
            K.gemm(x, ps.b[self.W], B, self.fpad, self.fin, 0, 0, out=out, out_f32=out_f32, bias=ps.p[self.Bn],
                   acct_flops=fl)
            if relu:
                K.relu_fwd(out)

    def backward(self, ps, dy, x, dx=None, bias_grad=True):
        B = x.shape[0]
        fl = 2 * B * self.fout * self.fin
        side = ps.side if dx is not None else None   # weight gradient beside the dgrad (ConvBN.backward)
        if side is not None:
            side.wait_stream(torch.cuda.current_stream())
            ps.side_used = True
        with torch.cuda.stream(side) if side is not None else _nullctx():
            if self.s_wg > 1:
                part = self.scratch.part[:self.s_wg * self.fpad * self.fin].view(self.s_wg, self.fpad, self.fin)
                K.gemm(dy, x, self.fpad, self.fin, B, 1, 1, out=part, splits=self.s_wg, acct_flops=fl)
                used = K.splits_used(B, self.s_wg)
                K.reduce_splits(part, used, self.fpad * self.fin, ps.g[self.W])
            else:
                # unsplit wgrad: 64-column N tiles so the (m, n) tiles fill the SMs
                K.gemm(dy, x, self.fpad, self.fin, B, 1, 1, out=ps.g[self.W], out_f32=True, acct_flops=fl,
                       max_bn=64)
            if bias_grad:
                K.col_sum(dy, B, self.fpad, self.fpad, ps.g[self.Bn])
            ps.grad_ready(self.W, self.Bn)
        if dx is not None:
            K.gemm(dy, ps.b[self.W], B, self.fin, self.fpad, 0, 1, out=dx, acct_flops=fl, max_bn=128)


class Net:
    """Common driver: loss head, Adam, buffers."""

    num_classes = 10
    in_channels = 3
    image = 32

    def __init__(self, seed=0):
        self.gen = torch.Generator().manual_seed(seed)
        self.ps = ParamStore()
        self.scratch = Scratch()
        self.lr, self.b1, self.b2, self.eps = 1e-3, 0.9, 0.999, 1e-8
        self.grad_scale = 1.0

    def build(self, batch, device="cuda", global_batch=None):
        self.batch = batch
        self.global_batch = global_batch or batch
        self.device = device
        self._build(batch, device)
        # fused classifier head (csrc/head.cu): one launch for the last Linear's forward, the loss
        # and its backward; CVB_UNFUSED_HEAD=1 keeps the gemm/softmax/col_sum launches
        h = self.head
        self.fused_head = (not _UNFUSED_HEAD and h.fpad == 16 and h.fin % 256 == 0 and h.fin <= 1024
                           and self.num_classes <= 16)
        if self.fused_head:
            self.scratch.part_floats = max(self.scratch.part_floats, K.head_workspace_floats(batch, h.fin))
        self.scratch.finalize(device)
        self.ps.finalize(device)
        fpad = self.head.fpad
        self.logits = torch.zeros(batch, fpad, dtype=F32, device=device)
        self.dlogits = torch.zeros(batch, fpad, dtype=BF16, device=device)
        self.row_loss = torch.zeros(batch, dtype=F32, device=device)
        self.loss = torch.zeros(1, dtype=F32, device=device)
        return self

    # models provide features(x) (everything before the head, writing head_in), features_backward(x,
    # fused) (everything after the head's dx), and the attributes head_in / head_dx / head_relu
    # (head_in is a ReLU output: mask dx) / prev_bias (Linear whose bias gradient = colsum(head_dx))
    prev_bias = None

    def forward(self, x):
        self.features(x)
        self.head.forward(self.ps, self.head_in, self.logits, out_f32=True)

    def backward(self, x):
        self.head.backward(self.ps, self.dlogits, self.head_in, self.head_dx)
        if self.head_relu:
            K.relu_bwd(self.head_dx, self.head_in)
        self.features_backward(x, False)

    def fwd_bwd(self, x, labels):
        """Forward, loss and backward of one step (gradients in ps.g32, loss in self.loss)."""
        ps = self.ps
        # wgrad/dgrad overlap on a side stream: single GPU, or data parallel with the collectives
        # captured inside the step graph (a segmented capture must not end a segment with
        # side-stream work outstanding)
        ps.side, ps.side_used = None, False
        if not _NO_OVERLAP and (ps.grad_hook is None or getattr(ps, "overlap_with_hook", False)) \
                and torch.cuda.is_available():
            if getattr(self, "_side", None) is None:
                self._side = torch.cuda.Stream()
            ps.side = self._side
        try:
            self._fwd_bwd(x, labels)
        finally:
            if ps.side_used:   # join only a stream that was forked from this one (graph capture)
                torch.cuda.current_stream().wait_stream(ps.side)
            ps.side, ps.side_used = None, False

    def _fwd_bwd(self, x, labels):
        if not self.fused_head:
            self.forward(x)
            self.loss_and_grad(labels)
            self.backward(x)
            return
        self.features(x)
        ps, h = self.ps, self.head
        pb = self.prev_bias
        K.head_train(self.head_in, ps.b[h.W], ps.p[h.Bn], labels, self.batch, self.num_classes,
                     1.0 / self.global_batch, self.logits, self.dlogits, self.row_loss, self.loss, ps.g[h.W],
                     ps.g[h.Bn], self.scratch.part, dx=self.head_dx, relu_mask=self.head_relu,
                     dprev_b=ps.g[pb.Bn] if pb is not None else None)
        ps.grad_ready(h.W, h.Bn)
        self.features_backward(x, True)

    def loss_and_grad(self, labels):
        K.softmax_xent(self.logits, self.batch, self.num_classes, labels, 1.0 / self.global_batch, self.row_loss,
                       self.loss, self.dlogits)

    def step(self, x, labels, allreduce=None):
        """One training step on a resident input tile (NHWC8 bf16) and int32 labels."""
        self.fwd_bwd(x, labels)
        if allreduce is not None:
            allreduce(self.ps.g32)
        self.optimizer_step()
        return self.loss

    def optimizer_step(self):
        K.adam_step(self.ps.p32, self.ps.g32, self.ps.m, self.ps.v, self.ps.pb, self.lr, self.b1, self.b2, self.eps,
                    step=0, grad_scale=self.grad_scale, step_dev=self.ps.step_dev, sched_dev=self.ps.sched,
                    skip_dev=self.ps.verdict_slot)
        self.ps.flip_all()   # next step's dgrad weights

    @property
    def num_params(self):
        return self.ps.logical


class SmallCNN(Net):
    """Paper-shaped CIFAR CNN: [conv3x3-BN-ReLU]x2, maxpool, [conv3x3-BN-ReLU]x2, maxpool,
    FC 4096-256 (ReLU), FC 256-10.  Input NHWC with channels padded 3 -> 8."""

    def __init__(self, seed=0, num_classes=10):
        super().__init__(seed)
        self.num_classes = num_classes
        ps, g = self.ps, self.gen
        self.c1 = ConvBN(ps, "conv1", 8, 32, 3, 1, 1, g, cin_real=3, need_dgrad=False)
        self.c2 = ConvBN(ps, "conv2", 32, 32, 3, 1, 1, g)
        self.c3 = ConvBN(ps, "conv3", 32, 64, 3, 1, 1, g)
        self.c4 = ConvBN(ps, "conv4", 64, 64, 3, 1, 1, g)
        self.fc1 = Linear(ps, "fc1", 8 * 8 * 64, 256, g)
        self.head = Linear(ps, "fc2", 256, num_classes, g)

    def _build(self, n, dev):
        S = self.scratch
        e = lambda *s: torch.empty(*s, dtype=BF16, device=dev)  # noqa: E731
        self.c1.build(n, 32, 32, S, dev)
        self.c2.build(n, 32, 32, S, dev)
        self.c3.build(n, 16, 16, S, dev)
        self.c4.build(n, 16, 16, S, dev)
        self.fc1.build(n, S)
        self.head.build(n, S)
        self.a1, self.a2, self.p1 = e(n, 32, 32, 32), e(n, 32, 32, 32), e(n, 16, 16, 32)
        self.a3, self.a4, self.p2 = e(n, 16, 16, 64), e(n, 16, 16, 64), e(n, 8, 8, 64)
        self.h = e(n, 256)
        self.dh, self.dp2 = e(n, 256), e(n, 8, 8, 64)
        self.da4, self.da3, self.dp1 = e(n, 16, 16, 64), e(n, 16, 16, 64), e(n, 16, 16, 32)
        self.da2, self.da1 = e(n, 32, 32, 32), e(n, 32, 32, 32)
        self.head_in, self.head_dx, self.head_relu, self.prev_bias = self.h, self.dh, True, self.fc1

    def features(self, x):
        ps = self.ps
        self.c1.forward(ps, x, self.a1)
        self.c2.forward(ps, self.a1, self.a2)
        K.maxpool_fwd(self.a2, 2, 2, 0, self.p1)
        self.c3.forward(ps, self.p1, self.a3)
        self.c4.forward(ps, self.a3, self.a4)
        K.maxpool_fwd(self.a4, 2, 2, 0, self.p2)
        flat = self.p2.view(self.batch, -1)
        self.fc1.forward(ps, flat, self.h, relu=True)

    def features_backward(self, x, fused):
        ps = self.ps
        flat = self.p2.view(self.batch, -1)
        # fused head: dh is already ReLU-masked and fc1's bias gradient already written
        self.fc1.backward(ps, self.dh, flat, self.dp2.view(self.batch, -1), bias_grad=not fused)
        K.maxpool_bwd(self.a4, self.dp2, 2, 2, 0, self.da4)
        self.c4.backward(ps, self.da4, self.a3, dx=self.da3)
        self.c3.backward(ps, self.da3, self.p1, dx=self.dp1)
        K.maxpool_bwd(self.a2, self.dp1, 2, 2, 0, self.da2)
        self.c2.backward(ps, self.da2, self.a1, dx=self.da1)
        self.c1.backward(ps, self.da1, x, dx=None)


class BasicBlock:
    def __init__(self, ps, name, cin, cout, stride, gen):
        self.c1 = ConvBN(ps, f"{name}.conv1", cin, cout, 3, stride, 1, gen, relu=True)
        self.c2 = ConvBN(ps, f"{name}.conv2", cout, cout, 3, 1, 1, gen, relu=True)  # relu after residual add
        self.down = None
        if stride != 1 or cin != cout:
            self.down = ConvBN(ps, f"{name}.down", cin, cout, 1, stride, 0, gen, relu=False)
        self.cin, self.cout = cin, cout

    def build(self, n, h, w, S, dev):
        oh, ow = self.c1.build(n, h, w, S, dev)
        self.c2.build(n, oh, ow, S, dev)
        e = lambda *s: torch.empty(*s, dtype=BF16, device=dev)  # noqa: E731
        self.o1, self.do1 = e(n, oh, ow, self.cout), e(n, oh, ow, self.cout)
        self.dres = e(n, oh, ow, self.cout)
        if self.down is not None:
            self.down.build(n, h, w, S, dev)
            self.sc = e(n, oh, ow, self.cout)
        return oh, ow

    def forward(self, ps, x, out):
        self.c1.forward(ps, x, self.o1)
        sc = x
        if self.down is not None:
            self.down.forward(ps, x, self.sc)
            sc = self.sc
        self.c2.forward(ps, self.o1, out, res=sc)

    def backward(self, ps, dout, x, out, dx):
        # out = relu(bn2(conv2(o1)) + sc): mask from `out`; the masked dout is the grad of sc
        if self.down is not None:
            self.c2.backward(ps, dout, self.o1, dx=self.do1, y=out, dres=self.dres)
            # 3x3 first (every output parity has taps), then the 1x1 shortcut accumulates
            self.c1.backward(ps, self.do1, x, dx=dx)
            self.down.backward(ps, self.dres, x, dx=dx, dx_accumulate=True)
        else:
            # identity shortcut: dx = masked dout (written by bn backward) + dgrad(conv1)
            self.c2.backward(ps, dout, self.o1, dx=self.do1, y=out, dres=dx)
            self.c1.backward(ps, self.do1, x, dx=dx, dx_accumulate=True)


class ResNet18(Net):
    """ResNet-18 for 32x32 inputs (3x3 stem, no max-pool), BasicBlock x [2,2,2,2]."""

    def __init__(self, seed=0, num_classes=10):
        super().__init__(seed)
        self.num_classes = num_classes
        ps, g = self.ps, self.gen
        self.stem = ConvBN(ps, "stem", 8, 64, 3, 1, 1, g, cin_real=3, need_dgrad=False)
        cfg = [(64, 64, 1), (64, 64, 1), (64, 128, 2), (128, 128, 1), (128, 256, 2), (256, 256, 1),
               (256, 512, 2), (512, 512, 1)]
        self.blocks = [BasicBlock(ps, f"layer{i // 2 + 1}.{i % 2}", ci, co, s, g) for i, (ci, co, s) in enumerate(cfg)]
        self.head = Linear(ps, "fc", 512, num_classes, g)

    def _build(self, n, dev):
        S = self.scratch
        e = lambda *s: torch.empty(*s, dtype=BF16, device=dev)  # noqa: E731
        self.stem.build(n, 32, 32, S, dev)
        self.x0 = e(n, 32, 32, 64)
        self.dx0 = e(n, 32, 32, 64)
        h = w = 32
        self.outs, self.douts = [], []
        for b in self.blocks:
            h, w = b.build(n, h, w, S, dev)
            self.outs.append(e(n, h, w, b.cout))
            self.douts.append(e(n, h, w, b.cout))
        self.final_hw = h * w
        self.pooled, self.dpooled = e(n, 512), e(n, 512)
        self.head.build(n, S)
        self.head_in, self.head_dx, self.head_relu = self.pooled, self.dpooled, False

    def features(self, x):
        ps = self.ps
        self.stem.forward(ps, x, self.x0)
        cur = self.x0
        for b, o in zip(self.blocks, self.outs):
            b.forward(ps, cur, o)
            cur = o
        K.gap_fwd(cur, self.batch, self.final_hw, 512, 512, self.pooled)

    def features_backward(self, x, fused):
        ps = self.ps
        K.gap_bwd(self.dpooled, self.batch, self.final_hw, 512, self.douts[-1])
        for i in range(len(self.blocks) - 1, -1, -1):
            b = self.blocks[i]
            xin = self.outs[i - 1] if i > 0 else self.x0
            dxin = self.douts[i - 1] if i > 0 else self.dx0
            b.backward(ps, self.douts[i], xin, self.outs[i], dxin)
        self.stem.backward(ps, self.dx0, x, dx=None)


class BNAct:
    """Pre-activation batch norm (+ReLU) over channels [0, C) of an NHWC buffer with a channel
    stride (DenseNet reads its concat buffer in place).  Backward accumulates the input
    gradient in fp32 (the concat gradient receives one contribution per later layer)."""

    def __init__(self, ps, name, C, relu=True):
        self.C, self.relu = C, relu
        self.G = ps.add(f"{name}.gamma", torch.ones(C))
        self.B = ps.add(f"{name}.beta", torch.zeros(C))

    def build(self, rows, scratch, device):
        self.rows = rows
        self.mean = torch.zeros(self.C, dtype=F32, device=device)
        self.rstd = torch.zeros(self.C, dtype=F32, device=device)
        self.run_mean = torch.zeros(self.C, dtype=F32, device=device)
        self.run_var = torch.ones(self.C, dtype=F32, device=device)
        scratch.bn_floats = max(scratch.bn_floats, K._lib_bound().cvb_bn_workspace_floats(rows, self.C))
        self.scratch = scratch

    def use_stats(self, mean, rstd):
        """Share precomputed per-channel batch statistics (DenseNet: every BN over a concat
        prefix sees the same per-channel mean/var -- computed once per produced slice)."""
        self.mean, self.rstd = mean, rstd
        self.shared = True

    def forward(self, ps, x, xcs, y, ycs, stats=True, pending=None):
        """pending = (off, n): the shared statistics of channels [off, off + n) are not computed
        yet -- they are computed in the same launch as the normalisation (DenseNet)."""
        if pending is not None:
            K.bn_forward_range(x, self.rows, self.C, xcs, self.scratch.bnws, self.mean, self.rstd, ps.p[self.G],
                               ps.p[self.B], y, ycs, pending[0], pending[1], relu=self.relu)
            return
        if stats and not getattr(self, "shared", False):
            K.bn_forward(x, self.rows, self.C, xcs, self.scratch.bnws, self.mean, self.rstd, ps.p[self.G],
                         ps.p[self.B], y, ycs, relu=self.relu, run_mean=self.run_mean, run_var=self.run_var)
            return
        K.bn_apply(x, self.rows, self.C, xcs, self.mean, self.rstd, ps.p[self.G], ps.p[self.B], y, ycs,
                   relu=self.relu)

    def backward(self, ps, dy, dycs, x, xcs, dx32, dx32cs, accumulate):
        K.bn_backward(dy, dycs, x, xcs, self.rows, self.C, self.mean, self.rstd, ps.p[self.G], ps.p[self.B],
                      self.scratch.bnws, ps.g[self.G], ps.g[self.B], relu=self.relu, dx32=dx32, dxcs=dx32cs,
                      accum32=accumulate)
        ps.grad_ready(self.G, self.B)


class Conv:
    """Convolution without a following BN (DenseNet's pre-activation units): bf16 output
    into a channel slice of the destination; backward = split-K wgrad + flipped-weight dgrad."""

    def __init__(self, ps, name, cin, cout, k, stride, pad, gen):
        self.cin, self.cout, self.k, self.s, self.pad = cin, cout, k, stride, pad
        bound = 1.0 / math.sqrt(cin * k * k)
        self.W = ps.add(f"{name}.w", _uniform(gen, (cout, k, k, cin), bound))
        if stride == 1:
            ps.want_flip(self.W)

    def build(self, n, h, w, scratch):
        self.n, self.h, self.w = n, h, w
        self.oh, self.ow = K.conv_out_hw(h, w, self.k, self.s, self.pad)
        self.flops = 2 * n * self.oh * self.ow * self.cout * self.k * self.k * self.cin
        count = self.cout * self.k * self.k * self.cin
        scratch.part_floats = max(scratch.part_floats, min(MAX_SPLITS * count, max(PART_CAP, 8 * count)))
        scratch.flip_elems = max(scratch.flip_elems, count)
        self.scratch = scratch
        return self.oh, self.ow

    def forward(self, ps, x, out, out_coff=0):
        K.conv2d_fwd(x, ps.b[self.W], self.s, self.pad, out=out, cin=self.cin, out_coff=out_coff,
                     acct_flops=self.flops)

    def backward(self, ps, dz, x, dx=None):
        count = self.cout * self.k * self.k * self.cin
        maxs = max(1, min(MAX_SPLITS, self.scratch.part.numel() // count))
        part, used = K.conv2d_wgrad_partials(dz, x, self.k, self.k, self.s, self.pad, cin=self.cin,
                                             part=self.scratch.part[:maxs * count].view(maxs, self.cout,
                                                                                        self.k * self.k * self.cin),
                                             acct_flops=self.flops)
        K.reduce_splits(part, used, count, ps.g[self.W])
        ps.grad_ready(self.W)
        if dx is not None:
            if self.W in ps.f:
                wt = ps.f[self.W]
            else:
                wt = self.scratch.flip[:count].view(self.cin, self.k, self.k, self.cout)
                K.weight_flip(ps.b[self.W], wt)
            K.conv2d_fwd(dz, wt, 1, self.k - 1 - self.pad, out=dx, out_hw=(self.h, self.w), acct_flops=self.flops)


class DenseLayer:
    """BN-ReLU-conv1x1(4g) -> BN-ReLU-conv3x3(g), output appended to the block buffer."""

    def __init__(self, ps, name, cin, growth, bn_size, gen):
        self.cin, self.growth, self.mid = cin, growth, bn_size * growth
        self.bn1 = BNAct(ps, f"{name}.norm1", cin)
        self.conv1 = Conv(ps, f"{name}.conv1", cin, self.mid, 1, 1, 0, gen)
        self.bn2 = BNAct(ps, f"{name}.norm2", self.mid)
        self.conv2 = Conv(ps, f"{name}.conv2", self.mid, growth, 3, 1, 1, gen)

    def build(self, n, h, w, S, dev):
        rows = n * h * w
        self.bn1.build(rows, S, dev)
        self.conv1.build(n, h, w, S)
        self.bn2.build(rows, S, dev)
        self.conv2.build(n, h, w, S)
        # deferred BN1 input gradient (DEFERRED_DX): the statistics pass's raw sums, kept apart
        # from the parameter gradients (those may be all-reduced in place before the gather)
        self.cg = torch.zeros(self.cin, dtype=F32, device=dev)
        self.cb = torch.zeros(self.cin, dtype=F32, device=dev)
        # kept for backward (no recompute): BN1/BN2 outputs and the 1x1 conv output
        self.z1 = torch.empty(n, h, w, self.mid, dtype=BF16, device=dev)
        self.y1 = torch.empty(n, h, w, self.cin, dtype=BF16, device=dev)
        self.y2 = torch.empty(n, h, w, self.mid, dtype=BF16, device=dev)

    def forward(self, ps, blk, y1=None, y2=None, pending=None, defer_stats=False):
        """pending: the previous layer's slice whose statistics this layer's BN1 computes in the
        same launch; defer_stats: leave this layer's slice statistics to the next BN over the block."""
        cs = blk.shape[-1]
        self.bn1.forward(ps, blk, cs, self.y1, self.cin, pending=pending)
        self.conv1.forward(ps, self.y1, self.z1)
        self.bn2.forward(ps, self.z1, self.mid, self.y2, self.mid)
        self.conv2.forward(ps, self.y2, blk, out_coff=self.cin)
        if not defer_stats:
            # batch statistics of the 32 new channels, shared by every later BN over this block
            m, r = self.slice_stats
            K.bn_stats(blk[..., self.cin:], self.bn1.rows, self.growth, cs, self.bn1.scratch.bnws, m, r)

    def gather_terms(self, ps, c0):
        """This layer's term of the deferred BN1 input gradient for channels from c0 on."""
        return (self.dy1_slot[..., c0:], self.cin, ps.p[self.bn1.G][c0:], ps.p[self.bn1.B][c0:], self.cg[c0:],
                self.cb[c0:])

    def backward(self, ps, blk, dblk32, y1, y2, dz2, dy2, dz1, dy1, later=None):
        cs = blk.shape[-1]
        rows = self.bn1.rows
        y1, y2 = self.y1, self.y2
        if later is None:
            # gradient of this layer's output slice is complete (later layers already added)
            K.cast_rows(dblk32[..., self.cin:], cs, dz2, self.growth, rows, self.growth)
        else:
            # deferred: the transition's gradient + every later layer's BN1 term, formed once
            m, r = self.slice_stats
            K.bn_gather_dx(blk[..., self.cin:], cs, rows, self.growth, m, r, [L.gather_terms(ps, self.cin) for L in later],
                           dz2, self.growth, base=dblk32[..., self.cin:], bcs=cs)
            dy1 = self.dy1_slot
        self.conv2.backward(ps, dz2, y2, dx=dy2)
        K.bn_backward(dy2, self.mid, self.z1, self.mid, rows, self.mid, self.bn2.mean, self.bn2.rstd,
                      ps.p[self.bn2.G], ps.p[self.bn2.B], self.bn2.scratch.bnws, ps.g[self.bn2.G], ps.g[self.bn2.B],
                      relu=True, dx=dz1, dxcs=self.mid)
        ps.grad_ready(self.bn2.G, self.bn2.B)
        self.conv1.backward(ps, dz1, y1, dx=dy1)
        if later is None:
            self.bn1.backward(ps, dy1, self.cin, blk, cs, dblk32, cs, accumulate=True)
        else:   # statistics pass only; the input gradient is gathered later
            b = self.bn1
            K.bn_backward(dy1, self.cin, blk, cs, b.rows, b.C, b.mean, b.rstd, ps.p[b.G], ps.p[b.B],
                          b.scratch.bnws, self.cg, self.cb, relu=b.relu)
            ps.g[b.G].copy_(self.cg)
            ps.g[b.B].copy_(self.cb)
            ps.grad_ready(b.G, b.B)


class DenseNet121(Net):
    """DenseNet-121-style (growth 32, blocks 6/12/24/16, bn_size 4, compression 0.5) for the
    medical config: 224x224x1 input (padded to 8 channels), 2 classes."""

    num_classes = 2
    in_channels = 1
    image = 224

    def __init__(self, seed=0, num_classes=2, blocks=(6, 12, 24, 16), growth=32, bn_size=4, init_ch=64):
        super().__init__(seed)
        self.num_classes = num_classes
        ps, g = self.ps, self.gen
        self.stem = ConvBN(ps, "features.conv0", 8, init_ch, 7, 2, 3, g, cin_real=1, need_dgrad=False)
        self.blocks, self.trans = [], []
        c = init_ch
        for bi, nl in enumerate(blocks):
            layers = [DenseLayer(ps, f"features.denseblock{bi + 1}.denselayer{li + 1}", c + li * growth, growth,
                                 bn_size, g) for li in range(nl)]
            self.blocks.append((c, c + nl * growth, layers))
            c = c + nl * growth
            if bi != len(blocks) - 1:
                t = (BNAct(ps, f"features.transition{bi + 1}.norm", c),
                     Conv(ps, f"features.transition{bi + 1}.conv", c, c // 2, 1, 1, 0, g))
                self.trans.append(t)
                c //= 2
        self.norm5 = BNAct(ps, "features.norm5", c)
        self.final_c = c
        self.head = Linear(ps, "classifier", c, num_classes, g)

    def _build(self, n, dev):
        S = self.scratch
        e = lambda *s: torch.empty(*s, dtype=BF16, device=dev)  # noqa: E731
        oh, ow = self.stem.build(n, 224, 224, S, dev)
        self.a0 = e(n, oh, ow, self.stem.cout)
        self.da0 = e(n, oh, ow, self.stem.cout)
        h, w = (oh + 2 - 3) // 2 + 1, (ow + 2 - 3) // 2 + 1
        self.pool_idx = torch.empty(n, h, w, self.stem.cout, dtype=torch.uint8, device=dev)   # stem max-pool arg-max
        self.geo, self.bufs, self.dbufs = [], [], []
        self.deferred = not os.environ.get("CVB_DENSE_ACCUM")   # A/B: per-layer fp32 accumulation
        self.merge_stats = not os.environ.get("CVB_DENSE_SLICE_STATS")   # A/B: separate slice-statistics launch
        self.bmean, self.brstd, self.ty = [], [], []
        ymax = 0
        for bi, (c0, c1, layers) in enumerate(self.blocks):
            bm = torch.zeros(c1, dtype=F32, device=dev)
            br = torch.zeros(c1, dtype=F32, device=dev)
            self.bmean.append(bm)
            self.brstd.append(br)
            for L in layers:
                L.build(n, h, w, S, dev)
                L.bn1.use_stats(bm[:L.cin], br[:L.cin])
                L.slice_stats = (bm[L.cin:L.cin + L.growth], br[L.cin:L.cin + L.growth])
            self.geo.append((h, w))
            self.bufs.append(e(n, h, w, c1))
            self.dbufs.append(torch.empty(n, h, w, c1, dtype=F32, device=dev))
            ymax = max(ymax, n * h * w * c1)
            if bi < len(self.trans):
                bn, conv = self.trans[bi]
                bn.build(n * h * w, S, dev)
                bn.use_stats(bm, br)
                conv.build(n, h, w, S)
                self.ty.append(e(n, h, w, c1))            # transition BN output, kept for backward
                h, w = h // 2, w // 2
        self.norm5.build(n * h * w, S, dev)
        self.norm5.use_stats(self.bmean[-1], self.brstd[-1])
        self.head.build(n, S)
        # shared scratch (largest use wins)
        mid = max(L.mid for _, _, ls in self.blocks for L in ls)
        rows_max = max(n * gh * gw for gh, gw in self.geo)
        self.y1 = e(ymax)
        self.y2 = e(rows_max * mid)
        self.dz2 = e(rows_max * 32)
        self.dy2 = e(rows_max * mid)
        self.dz1 = e(rows_max * mid)
        self.dy1 = e(ymax)
        self.t = e(ymax // 2)
        self.dt = e(ymax // 2)
        self.y5 = e(n * h * w * self.final_c)
        self.dy5 = e(n * h * w * self.final_c)
        self.final_hw = h * w
        self.pooled, self.dpooled = e(n, self.final_c), e(n, self.final_c)
        self.head_in, self.head_dx, self.head_relu = self.pooled, self.dpooled, False
        self.dcast = e(ymax)
        if self.deferred:   # every layer's dY1 stays alive until its block's gradients are gathered
            need = 0
            for bi, (c0, c1, layers) in enumerate(self.blocks):
                gh, gw = self.geo[bi]
                need = max(need, sum(n * gh * gw * L.cin for L in layers))
            self.dy1_store = e(need)
            for bi, (c0, c1, layers) in enumerate(self.blocks):
                gh, gw = self.geo[bi]
                off = 0
                for L in layers:
                    cnt = n * gh * gw * L.cin
                    L.dy1_slot = self.dy1_store[off:off + cnt].view(n, gh, gw, L.cin)
                    off += cnt

    def _v(self, buf, *shape):
        return buf[:math.prod(shape)].view(*shape)

    def features(self, x):
        ps, n = self.ps, self.batch
        self.stem.forward(ps, x, self.a0)
        c0 = self.stem.cout
        K.maxpool_fwd(self.a0, 3, 2, 1, self.bufs[0][..., :c0], idx=self.pool_idx)
        h, w = self.geo[0]
        K.bn_stats(self.bufs[0], n * h * w, c0, self.bufs[0].shape[-1], self.scratch.bnws, self.bmean[0][:c0],
                   self.brstd[0][:c0])
        for bi, (c0, c1, layers) in enumerate(self.blocks):
            h, w = self.geo[bi]
            blk = self.bufs[bi]
            pend = None
            for L in layers:
                # the newest slice's statistics are computed by the next BN over the block, in
                # the same launch as its normalisation (no separate statistics launch)
                L.forward(ps, blk, pending=pend, defer_stats=self.merge_stats)
                pend = (L.cin, L.growth) if self.merge_stats else None
            if bi < len(self.trans):
                bn, conv = self.trans[bi]
                y = self.ty[bi]
                bn.forward(ps, blk, c1, y, c1, pending=pend)
                t = self._v(self.t, n, h, w, c1 // 2)
                conv.forward(ps, y, t)
                nxt = self.bufs[bi + 1]
                K.avgpool_fwd(t, n, h, w, c1 // 2, c1 // 2, 2, nxt, nxt.shape[-1])
                K.bn_stats(nxt, n * (h // 2) * (w // 2), c1 // 2, nxt.shape[-1], self.scratch.bnws,
                           self.bmean[bi + 1][:c1 // 2], self.brstd[bi + 1][:c1 // 2])
        h, w = self.geo[-1]
        c = self.final_c
        self.norm5.forward(ps, self.bufs[-1], c, self._v(self.y5, n, h, w, c), c, pending=pend)
        K.gap_fwd(self._v(self.y5, n, h, w, c), n, h * w, c, c, self.pooled)

    def features_backward(self, x, fused):
        ps, n = self.ps, self.batch
        c = self.final_c
        h, w = self.geo[-1]
        dy5 = self._v(self.dy5, n, h, w, c)
        K.gap_bwd(self.dpooled, n, h * w, c, dy5)
        self.norm5.backward(ps, dy5, c, self.bufs[-1], c, self.dbufs[-1], c, accumulate=False)
        for bi in range(len(self.blocks) - 1, -1, -1):
            c0, c1, layers = self.blocks[bi]
            h, w = self.geo[bi]
            blk, dblk = self.bufs[bi], self.dbufs[bi]
            if bi < len(self.trans):
                # transition: its input gradient initialises this block's fp32 concat gradient
                bn, conv = self.trans[bi]
                nxt_d = self.dbufs[bi + 1]
                oh, ow = h // 2, w // 2
                dp = self._v(self.dcast, n, oh, ow, c1 // 2)
                K.cast_rows(nxt_d, nxt_d.shape[-1], dp, c1 // 2, n * oh * ow, c1 // 2)
                dt = self._v(self.dt, n, h, w, c1 // 2)
                K.avgpool_bwd(dp, n, h, w, c1 // 2, 2, dt, c1 // 2)
                y = self.ty[bi]
                dy = self._v(self.dy1, n, h, w, c1)
                conv.backward(ps, dt, y, dx=dy)
                bn.backward(ps, dy, c1, blk, c1, dblk, c1, accumulate=False)
            for li in range(len(layers) - 1, -1, -1):
                L = layers[li]
                later = [layers[j] for j in range(len(layers) - 1, li, -1)] if self.deferred else None
                L.backward(ps, blk, dblk, self._v(self.y1, n, h, w, L.cin), self._v(self.y2, n, h, w, L.mid),
                           self._v(self.dz2, n, h, w, L.growth), self._v(self.dy2, n, h, w, L.mid),
                           self._v(self.dz1, n, h, w, L.mid), self._v(self.dy1, n, h, w, L.cin), later=later)
            if self.deferred:   # the block input's gradient: the transition's term + every layer's
                K.bn_gather_dx(blk, blk.shape[-1], n * h * w, c0, self.bmean[bi][:c0], self.brstd[bi][:c0],
                               [layers[j].gather_terms(ps, 0) for j in range(len(layers) - 1, -1, -1)],
                               dblk, dblk.shape[-1], base=dblk, bcs=dblk.shape[-1])
        # stem: max-pool backward from the first 64 channels of block 1's gradient
        h, w = self.geo[0]
        d0 = self._v(self.dcast, n, h, w, self.stem.cout)
        K.cast_rows(self.dbufs[0], self.dbufs[0].shape[-1], d0, self.stem.cout, n * h * w, self.stem.cout)
        K.maxpool_bwd(self.a0, d0, 3, 2, 1, self.da0, idx=self.pool_idx)
        self.stem.backward(ps, self.da0, x, dx=None)


MODELS = {"small_cnn": SmallCNN, "resnet18": ResNet18, "densenet121": DenseNet121}


def make_model(name, seed=0, **kw):
    return MODELS[name](seed=seed, **kw)

"""PyTorch-CPU restatement of the CNN training step -- TEST INFRASTRUCTURE ONLY.

PARITY UNPINNED AGAINST THE REFERENCE: the reference (covault) has no CNN code at all --
its trainer is the logistic toy in pkg/src/covault/workload.py:48-71, and the CIFAR CNN /
medical models exist only as prose in PAPER.md:441-443 and :475-477.  This module is the
builder-written CPU oracle for those models, used only by tests/, smoke()
and bench.py's CPU baseline.

It follows the numeric contract of paper_2103_16898_b200/nets.py exactly:
  * conv / FC operands are the bf16 roundings of the fp32 master weights,
  * every stored activation is rounded to bf16 (RB) and so is every activation gradient
    (RB rounds its incoming gradient too), accumulation is fp32,
  * logits are fp32, dlogits are rounded to bf16 (RBG),
  * BN uses batch statistics (biased variance) in fp32, running stats with momentum 0.1,
  * Adam = torch.optim.Adam(lr=1e-3, betas=(0.9, 0.999), eps=1e-8) on fp32 masters.
With full fp32 (``emulate_bf16=False``) it is the plain fp32 reference used for the looser
bf16-vs-fp32 tolerance.
"""
from __future__ import annotations

import torch
import torch.nn.functional as F


class _RB(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x):
        return x.to(torch.bfloat16).float()

    @staticmethod
    def backward(ctx, g):
        return g.to(torch.bfloat16).float()


class _RBG(torch.autograd.Function):
    """identity forward, bf16-rounded gradient"""

    @staticmethod
    def forward(ctx, x):
        return x.clone()

    @staticmethod
    def backward(ctx, g):
        return g.to(torch.bfloat16).float()


class Rounding:
    def __init__(self, emulate_bf16=True):
        self.on = emulate_bf16

    def rb(self, x):
        return _RB.apply(x) if self.on else x

    def rbg(self, x):
        return _RBG.apply(x) if self.on else x

    def w(self, p):
        return p.to(torch.bfloat16).float() if self.on else p


def nhwc_conv_weight(w_nhwc, cin_real=None):
    """[co][kh][kw][ci] -> torch [co][ci][kh][kw] (drop padded input channels)."""
    w = w_nhwc.permute(0, 3, 1, 2)
    if cin_real is not None:
        w = w[:, :cin_real]
    return w.contiguous()


class RefModel(torch.nn.Module):
    """Holds fp32 leaf parameters keyed like nets.ParamStore (NHWC weight layout)."""

    def __init__(self, state: dict, emulate_bf16=True):
        super().__init__()
        self.R = Rounding(emulate_bf16)
        self.names = list(state.keys())
        self.params = torch.nn.ParameterDict({k.replace(".", "__"): torch.nn.Parameter(v.clone().float())
                                              for k, v in state.items()})
        self.running = {}
        # mask matching (tests/cnn_parity.py): ReLU masks and 2x2 max-pool arg-max positions
        # taken from the GPU's own forward pass, so fp32-summation-order noise cannot toggle a
        # near-zero pre-activation or a near-tie window between the two runs; the oracle still
        # computes every value itself
        self.forced_relu, self.forced_pool = {}, {}

    def force(self, relu_masks=None, pool_argmax=None):
        self.forced_relu = dict(relu_masks or {})
        self.forced_pool = dict(pool_argmax or {})

    def relu(self, y, site):
        m = self.forced_relu.get(site)
        return F.relu(y) if m is None else y * m

    def maxpool2(self, x, site):
        idx = self.forced_pool.get(site)
        if idx is None:
            return F.max_pool2d(x, 2)
        n, c, h, w = x.shape
        win = x.reshape(n, c, h // 2, 2, w // 2, 2).permute(0, 1, 2, 4, 3, 5).reshape(n, c, h // 2, w // 2, 4)
        return win.gather(-1, idx.unsqueeze(-1)).squeeze(-1)

    def P(self, name):
        return self.params[name.replace(".", "__")]

    def conv_bn(self, x, name, stride, pad, relu=True, res=None, cin_real=None):
        R = self.R
        w = self.P(f"{name}.w")
        wt = nhwc_conv_weight(_bf16_param(w) if R.on else w, cin_real)
        z = R.rb(F.conv2d(x, wt, stride=stride, padding=pad))
        rm = self.running.setdefault(name + ".rm", torch.zeros(z.shape[1]))
        rv = self.running.setdefault(name + ".rv", torch.ones(z.shape[1]))
        y = F.batch_norm(z, rm, rv, self.P(f"{name}.gamma"), self.P(f"{name}.beta"), training=True, momentum=0.1,
                         eps=1e-5)
        if res is not None:
            y = y + res
        if relu:
            y = self.relu(y, name)
        return R.rb(y)

    def linear(self, x, name, fout, out_f32=False, relu=False):
        R = self.R
        w = self.P(f"{name}.w")[:fout]
        b = self.P(f"{name}.b")[:fout]
        wb = _bf16_param(w) if R.on else w
        y = x @ wb.t() + b
        if relu:
            y = self.relu(y, name)
        return y if out_f32 else R.rb(y)


def _bf16_param(w):
    """bf16 rounding of a parameter with a straight-through (unrounded) gradient: the GPU
    accumulates weight gradients in fp32 against the bf16 operand copy."""
    return w + (w.detach().to(torch.bfloat16).float() - w.detach())


class SmallCNNRef(RefModel):
    def forward(self, x):           # x: NCHW fp32 (bf16 values), 3 channels
        R = self.R
        a = self.conv_bn(x, "conv1", 1, 1, cin_real=3)
        a = self.conv_bn(a, "conv2", 1, 1)
        a = self.maxpool2(a, "pool1")
        a = self.conv_bn(a, "conv3", 1, 1)
        a = self.conv_bn(a, "conv4", 1, 1)
        a = self.maxpool2(a, "pool2")
        flat = R.rb(a.permute(0, 2, 3, 1).reshape(a.shape[0], -1))   # NHWC flatten order
        h = self.linear(flat, "fc1", 256, relu=True)
        return self.linear(h, "fc2", self.num_classes, out_f32=True)

    num_classes = 10


class ResNet18Ref(RefModel):
    cfg = [(64, 64, 1), (64, 64, 1), (64, 128, 2), (128, 128, 1), (128, 256, 2), (256, 256, 1), (256, 512, 2),
           (512, 512, 1)]
    num_classes = 10

    def forward(self, x):
        R = self.R
        a = self.conv_bn(x, "stem", 1, 1, cin_real=3)
        for i, (ci, co, s) in enumerate(self.cfg):
            nm = f"layer{i // 2 + 1}.{i % 2}"
            o1 = self.conv_bn(a, f"{nm}.conv1", s, 1)
            sc = a
            if s != 1 or ci != co:
                sc = self.conv_bn(a, f"{nm}.down", s, 0, relu=False)
            a = self.conv_bn(o1, f"{nm}.conv2", 1, 1, res=sc)
        pooled = R.rb(a.mean(dim=(2, 3)))
        return self.linear(pooled, "fc", self.num_classes, out_f32=True)


class DenseNet121Ref(RefModel):
    """DenseNet-121-style, 1-channel 224x224 stem, 2 classes (nets.DenseNet121).  Rounding
    points: BN outputs, conv outputs and pool outputs are bf16; the concat gradient is fp32
    (autograd sums the per-layer contributions) and is rounded where the GPU casts it."""

    num_classes = 2
    blocks = (6, 12, 24, 16)
    growth, bn_size, init_ch = 32, 4, 64

    def bn_relu(self, x, name, relu=True):
        rm = self.running.setdefault(name + ".rm", torch.zeros(x.shape[1]))
        rv = self.running.setdefault(name + ".rv", torch.ones(x.shape[1]))
        y = F.batch_norm(x, rm, rv, self.P(f"{name}.gamma"), self.P(f"{name}.beta"), training=True, momentum=0.1,
                         eps=1e-5)
        return self.R.rb(F.relu(y) if relu else y)

    def conv(self, x, name, stride, pad):
        w = self.P(f"{name}.w")
        wt = nhwc_conv_weight(_bf16_param(w) if self.R.on else w)
        return self.R.rb(F.conv2d(x, wt, stride=stride, padding=pad))

    def forward(self, x):
        R = self.R
        a = self.conv_bn(x, "features.conv0", 2, 3, cin_real=1)
        a = R.rb(F.max_pool2d(a, 3, 2, 1))
        feats = [a]
        for bi, nl in enumerate(self.blocks):
            for li in range(nl):
                nm = f"features.denseblock{bi + 1}.denselayer{li + 1}"
                cat = torch.cat(feats, dim=1)
                y1 = self.bn_relu(cat, f"{nm}.norm1")
                z1 = self.conv(y1, f"{nm}.conv1", 1, 0)
                y2 = self.bn_relu(z1, f"{nm}.norm2")
                feats.append(self.conv(y2, f"{nm}.conv2", 1, 1))
            cat = torch.cat(feats, dim=1)
            if bi != len(self.blocks) - 1:
                y = self.bn_relu(cat, f"features.transition{bi + 1}.norm")
                t = self.conv(y, f"features.transition{bi + 1}.conv", 1, 0)
                feats = [R.rb(F.avg_pool2d(t, 2))]
        y5 = self.bn_relu(cat, "features.norm5")
        pooled = R.rb(y5.mean(dim=(2, 3)))
        return self.linear(pooled, "classifier", self.num_classes, out_f32=True)


REF_MODELS = {"small_cnn": SmallCNNRef, "resnet18": ResNet18Ref, "densenet121": DenseNet121Ref}


def normalise_records(records_u8: torch.Tensor, c: int, h: int, w: int, mean, std, emulate_bf16=True):
    """uint8 records [n][1+c*h*w] -> (NCHW fp32 input, int64 labels), same arithmetic as
    csrc/loader.cu and the fused decrypt-decode: v = fma(x, 1/(255*std), -mean/std) rounded once
    to fp32 (x * scale is exact in fp64 for 8-bit x and the sum of two ~unit-range values fits
    53 bits, so the fp64 expression rounded to fp32 is the fused multiply-add), then bf16."""
    labels = records_u8[:, 0].long()
    px = records_u8[:, 1:].double().view(-1, c, h, w)
    import numpy as np

    f32 = np.float32   # the per-channel factors are computed in fp32 on the host side of the kernels
    scale = torch.tensor([f32(1.0) / (f32(255.0) * f32(s)) for s in std], dtype=torch.float32).view(1, c, 1, 1)
    shift = torch.tensor([-f32(m) / f32(s) for m, s in zip(mean, std)], dtype=torch.float32).view(1, c, 1, 1)
    x = (px * scale.double() + shift.double()).float()
    if emulate_bf16:
        x = x.to(torch.bfloat16).float()
    return x, labels


class RefTrainer:
    def __init__(self, name, state, emulate_bf16=True, lr=1e-3):
        self.model = REF_MODELS[name](state, emulate_bf16)
        self.opt = torch.optim.Adam(self.model.parameters(), lr=lr, betas=(0.9, 0.999), eps=1e-8, foreach=False)

    def load(self, state, exp_avg=None, exp_avg_sq=None, step=0):
        """Teacher forcing: start the next step from the given weights and Adam state (the GPU's
        pre-step state), so one step is compared on identical parameters."""
        with torch.no_grad():
            for k, p in self.model.params.items():
                name = k.replace("__", ".")
                p.copy_(state[name])
                if step > 0:
                    st = self.opt.state[p]
                    st["step"] = torch.tensor(float(step))
                    st["exp_avg"] = exp_avg[name].clone().float()
                    st["exp_avg_sq"] = exp_avg_sq[name].clone().float()
                else:
                    self.opt.state.pop(p, None)

    def step(self, x, labels):
        self.opt.zero_grad(set_to_none=False)
        logits = self.model(x)
        logits = self.model.R.rbg(logits)
        loss = F.cross_entropy(logits, labels)
        loss.backward()
        grads = {n: p.grad.detach().clone() for n, p in self.model.params.items()}
        self.opt.step()
        return float(loss.detach()), grads

    def state(self):
        return {k.replace("__", "."): v.detach().clone() for k, v in self.model.params.items()}

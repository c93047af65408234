"""Layer tables of the BASELINE.json configurations.

The reference network is purely sequential (net.hpp:13-15), so "ResNet-shaped"
means per-layer captures with these shapes fed to the step, not a ResNet
forward pass.  Each entry is a layer of the optimizer step:
  ("conv", c_in, c_out, k, stride, pad, h_in, w_in)  -> Kronecker layer
  ("fc", d_in, d_out)                                -> Kronecker layer
  ("bn", channels, hw)                               -> unit-wise BN layer
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Tuple


@dataclass(frozen=True)
class Layer:
    kind: str            # "conv" | "fc" | "bn"
    c_in: int = 0
    c_out: int = 0
    k: int = 1
    stride: int = 1
    pad: int = 0
    h_in: int = 1
    w_in: int = 1

    @property
    def h_out(self):
        return (self.h_in + 2 * self.pad - self.k) // self.stride + 1 if self.kind == "conv" else 1

    @property
    def w_out(self):
        return (self.w_in + 2 * self.pad - self.k) // self.stride + 1 if self.kind == "conv" else 1

    @property
    def hw(self):
        return self.h_out * self.w_out

    @property
    def a(self):
        return self.c_in * self.k * self.k if self.kind == "conv" else self.c_in

    @property
    def g(self):
        return self.c_out


def conv(c_in, c_out, k, stride, h):
    return Layer("conv", c_in, c_out, k, stride, (k - 1) // 2 if k > 1 else 0, h, h)


def bn(c, hw=1):
    return Layer("bn", c, c, 1, 1, 0, hw, 1)


def fc(d_in, d_out):
    return Layer("fc", d_in, d_out)


def resnet50() -> List[Layer]:
    """torchvision v1.5 (stride on the 3x3), 224x224: 53 conv + 53 BN + FC."""
    L = [conv(3, 64, 7, 2, 224), bn(64)]
    h, c_in = 56, 64
    for width, blocks, stride in [(64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)]:
        out = width * 4
        for b in range(blocks):
            s = stride if b == 0 else 1
            L += [conv(c_in, width, 1, 1, h), bn(width)]
            L += [conv(width, width, 3, s, h), bn(width)]
            h2 = (h + 2 - 3) // s + 1
            L += [conv(width, out, 1, 1, h2), bn(out)]
            if b == 0:
                L += [conv(c_in, out, 1, s, h), bn(out)]
            c_in, h = out, h2
    L.append(fc(2048, 1000))
    return L


def resnet18_cifar() -> List[Layer]:
    """CIFAR ResNet-18, 32x32: 20 conv + 20 BN + FC (4,800 BN channels)."""
    L = [conv(3, 64, 3, 1, 32), bn(64)]
    h, c_in = 32, 64
    for width, stride in [(64, 1), (128, 2), (256, 2), (512, 2)]:
        for b in range(2):
            s = stride if b == 0 else 1
            h2 = (h + 2 - 3) // s + 1
            L += [conv(c_in, width, 3, s, h), bn(width)]
            L += [conv(width, width, 3, 1, h2), bn(width)]
            if b == 0 and (s != 1 or c_in != width):
                L += [conv(c_in, width, 1, s, h), bn(width)]
            c_in, h = width, h2
    L.append(fc(512, 10))
    return L


def mlp() -> List[Layer]:
    """3-layer MLP 784-256-256-10 (BASELINE config 1)."""
    return [fc(784, 256), fc(256, 256), fc(256, 10)]


CONFIGS = {
    "mlp": (mlp, 128, "3-layer MLP 784-256-256-10, batch 128"),
    "resnet18": (resnet18_cifar, 128, "ResNet-18 CIFAR 32x32, batch 128/GPU"),
    "resnet50": (resnet50, 32, "ResNet-50 224x224, batch 32/GPU"),
}


def kron_layers(layers):
    return [l for l in layers if l.kind != "bn"]


def flops(layers, batch) -> Tuple[float, float, float]:
    """(F_factor per GPU, F_inverse total, F_precondition total), SURVEY.md §8d."""
    ff = fi = fp = 0.0
    for l in kron_layers(layers):
        K = batch * l.hw
        a, g = l.a, l.g
        ff += (a * (a + 1) + g * (g + 1)) * K
        fi += a ** 3 + g ** 3
        fp += 2 * g * g * a + 2 * g * a * a
    return ff, fi, fp


def capture_bytes(layers, batch) -> int:
    b = 0
    for l in layers:
        if l.kind == "bn":
            b += 2 * batch * l.c_out * 4
        else:
            b += batch * (l.a + l.g) * l.hw * 4
    return b

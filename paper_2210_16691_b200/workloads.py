"""The BASELINE.json workloads and the schedule each one
runs with, shared by bench.py and the scale-parity tests so the tests check
exactly the kernels and schedules the bench times.

C1  fp16 GEMM 512^3, the reference's own schedule script (tile 128x128x32, 2+2)
C2  BERT-base layer GEMMs, M = 4096 tokens, (N, K) in {768, 3072}
C3  attention batched GEMMs, batch*heads = 192, seq 512, head_dim 64
C4  ResNet-50 v1.5 implicit-GEMM convs, batch 256, NHWC
C5  square bf16 GEMMs n = 4096 .. 16384, M-sharded across ranks
"""
from __future__ import annotations

from dataclasses import dataclass

BERT_GEMMS = [  # (name, M, N, K): Q/K/V fused into one launch (weights side by side)
    ("qkv_proj", 4096, 2304, 768), ("o_proj", 4096, 768, 768), ("ffn1", 4096, 3072, 768),
    ("ffn2", 4096, 768, 3072),
]
BERT_GEMMS_UNFUSED = [
    ("q_proj", 4096, 768, 768), ("k_proj", 4096, 768, 768), ("v_proj", 4096, 768, 768),
    ("o_proj", 4096, 768, 768), ("ffn1", 4096, 3072, 768), ("ffn2", 4096, 768, 3072),
]

BMM_BATCH = 192
BMM_ATTENTION = [("qk_t", 512, 512, 64), ("pv", 512, 64, 512)]  # (name, M, N, K) per batch entry

SQUARES = (4096, 8192, 12288, 16384)
SQUARE_GRANULE = 256  # M-shard granule: one CTA-pair tile row

RESNET_BATCH = 256
# (name, H_in, C, K, R, stride, pad, repeats in ResNet-50 v1.5)
RESNET50_CONVS = [
    ("conv1_7x7s2_3_64", 224, 3, 64, 7, 2, 3, 1),  # the stem kernel: NHWC4 input (zero channel 3)
    ("l1_1x1_64_64", 56, 64, 64, 1, 1, 0, 1), ("l1_3x3_64_64", 56, 64, 64, 3, 1, 1, 3),
    ("l1_1x1_64_256", 56, 64, 256, 1, 1, 0, 4), ("l1_1x1_256_64", 56, 256, 64, 1, 1, 0, 2),
    ("l2_1x1_256_128", 56, 256, 128, 1, 1, 0, 1), ("l2_3x3s2_128", 56, 128, 128, 3, 2, 1, 1),
    ("l2_3x3_128", 28, 128, 128, 3, 1, 1, 3), ("l2_1x1_128_512", 28, 128, 512, 1, 1, 0, 4),
    ("l2_ds_256_512", 56, 256, 512, 1, 2, 0, 1), ("l2_1x1_512_128", 28, 512, 128, 1, 1, 0, 3),
    ("l3_1x1_512_256", 28, 512, 256, 1, 1, 0, 1), ("l3_3x3s2_256", 28, 256, 256, 3, 2, 1, 1),
    ("l3_3x3_256", 14, 256, 256, 3, 1, 1, 5), ("l3_1x1_256_1024", 14, 256, 1024, 1, 1, 0, 6),
    ("l3_ds_512_1024", 28, 512, 1024, 1, 2, 0, 1), ("l3_1x1_1024_256", 14, 1024, 256, 1, 1, 0, 5),
    ("l4_1x1_1024_512", 14, 1024, 512, 1, 1, 0, 1), ("l4_3x3s2_512", 14, 512, 512, 3, 2, 1, 1),
    ("l4_3x3_512", 7, 512, 512, 3, 1, 1, 2), ("l4_1x1_512_2048", 7, 512, 2048, 1, 1, 0, 3),
    ("l4_ds_1024_2048", 14, 1024, 2048, 1, 2, 0, 1), ("l4_1x1_2048_512", 7, 2048, 512, 1, 1, 0, 2),
]


@dataclass(frozen=True)
class ConvLayer:
    name: str
    H: int          # input height = width
    C: int          # logical input channels
    K: int
    R: int          # filter height = width
    stride: int
    pad: int
    repeats: int

    @property
    def P(self) -> int:
        return (self.H + 2 * self.pad - self.R) // self.stride + 1

    @property
    def stem(self) -> bool:
        """The stem kernel (csrc/stem_sm100.cu): C <= 4 stored as 4 channels,
        horizontal stride 2 (ResNet-50 conv1)."""
        return self.C <= 4 and self.stride == 2 and self.H % 16 == 0 and self.K % 64 == 0 and self.K <= 256

    @property
    def gemm(self) -> bool:
        """1x1, stride 1, no padding: the conv is a plain GEMM and runs on the GEMM
        kernels (CTA-pair tiles included)."""
        return self.R == 1 and self.stride == 1 and self.pad == 0

    @property
    def window(self) -> bool:
        """The window mode of the resident-filter kernel: C = 64, stride 1, a
        spatial filter whose K x R x S x 64 filter fits (ResNet-50 l1 3x3)."""
        return self.C == 64 and self.stride == 1 and self.R > 1 and self.R * self.R * self.K * 128 <= 80 * 1024

    @property
    def stream(self) -> bool:
        """The window mode with a streamed filter: C = 64 x CB > 64, K <= 128, stride 1, a spatial
        filter, a map tall enough for the window tiles (ResNet-50 l2 3x3)."""
        q = self.P
        wp = 16
        while wp < q + self.R - 1:
            wp *= 2
        return (self.C % 64 == 0 and self.C > 64 and self.K <= 128 and self.stride == 1 and self.R > 1
                and wp <= 128 and self.P >= 128 // wp)

    @property
    def Cs(self) -> int:
        """Stored channels: 4 on the stem kernel, else NHWC rows padded to the
        16-byte TMA granule."""
        return 4 if self.stem else -(-self.C // 8) * 8

    @property
    def halo(self) -> bool:
        """The input is stored with its zero-padding halo (one TMA box per
        filter row, R*64 reduction elements) when a filter row's S*C taps fit
        one 128-byte row (the 1x1 / C = 64 layer; pad 0, so no halo bytes)."""
        return not self.stem and self.R * self.Cs <= 64

    def gemm_k(self) -> int:
        """Reduction length of the GEMM view the kernel runs."""
        if self.stem:  # R filter rows x pair groups (pad % 2 + S taps, rounded to an even count of pairs) x 8
            t = (self.pad % 2 + self.R + 1) // 2
            return self.R * ((t + 1) // 2 * 2) * 8
        return self.R * 64 if self.halo else self.R * self.R * self.Cs

    def flops(self, n: int) -> float:
        """2*(N*P*Q)*K*(C*R*S) at the logical channel count."""
        return 2.0 * n * self.P * self.P * self.K * self.R * self.R * self.C

    def compulsory_bytes(self, n: int, elem: int = 2) -> int:
        """Bytes the layer must move: the input pixels the filter windows touch
        (a strided 1x1 conv reads only every stride-th row and column), the
        filter, and the output."""
        if self.R == 1 and self.stride > 1:
            touched = n * self.P * self.P * self.C
        else:
            touched = n * self.H * self.H * self.C
        return elem * (touched + self.K * self.R * self.R * self.C + n * self.P * self.P * self.K)


CONV_LAYERS = [ConvLayer(*row) for row in RESNET50_CONVS]


def conv_gemm_desc(alcop, layer: ConvLayer, nimg: int, in_dtype=None, out_dtype=None):
    """The conv's GEMM view (M = N*P*Q, N = K, K = R*S*C) the schedule model ranks."""
    return alcop.gemm_desc(nimg * layer.P * layer.P, layer.K, layer.gemm_k(), 1,
                           alcop.BF16 if in_dtype is None else in_dtype,
                           alcop.BF16 if out_dtype is None else out_dtype, alcop.B_NK)


def conv_desc(alcop, layer: ConvLayer, nimg: int, in_dtype=None, out_dtype=None):
    """The ABI descriptor of the layer as the bench stores it (NHWC, C padded to
    Cs; the stem's input carries its zero-padding halo)."""
    d = alcop.conv_desc(nimg, layer.H, layer.H, layer.Cs, layer.K, layer.R, layer.R, (layer.stride, layer.stride),
                        (layer.pad, layer.pad), alcop.BF16 if in_dtype is None else in_dtype,
                        alcop.BF16 if out_dtype is None else out_dtype)
    d.x_halo = 1 if layer.halo else 0
    return d


def conv_schedule(alcop, layer: ConvLayer, nimg: int):
    """The schedule the bench runs the layer with (alcop_choose_conv_schedule)."""
    return alcop.choose_conv_schedule(conv_desc(alcop, layer, nimg))


def square_schedule(alcop, m: int, n: int):
    """The schedule the bench runs an m x n x n square shard with (the model's pick)."""
    return alcop.choose_schedule(alcop.gemm_desc(m, n, n, 1, alcop.BF16, alcop.BF16, alcop.B_KN))

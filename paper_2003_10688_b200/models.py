"""BASELINE.json model configs built with the reference-style GraphBuilder.

Architectures follow torchvision (ResNet-18/50, DenseNet-121, MobileNet-V2) expressed in the
reference IR (Conv2d / BatchNorm2d / ReLU / MaxPool2d / AvgPool2d / Add / GlobalAvgPool /
Linear / Softmax / CrossEntropyLoss) plus the Concat and ReLU6 extensions. Weights are
random-initialised (no network for checkpoints); the input is "x" [B,3,H,W] and, for training
graphs, one-hot labels "t" [B, classes].
"""
from __future__ import annotations

from .graph import GraphBuilder, ModelGraph, meta_nc, meta_nchw


def _head(b: GraphBuilder, feat: str, c: int, classes: int, train: bool):
    fc = b.linear("fc", feat, c, classes)
    prob = b.softmax("prob", fc)
    if train:
        b.input("t", meta_nc(0, classes))
        return b.done([b.ce("loss", prob, "t")])
    return b.done([prob])


def small_cnn(classes: int = 10, hw: int = 32, train: bool = False, seed: int = 7) -> ModelGraph:
    """Config C1: 2x (conv-BN-ReLU-maxpool) + linear (BASELINE.json configs[0])."""
    b = GraphBuilder(seed)
    b.input("x", meta_nchw(0, 3, hw, hw))
    x = "x"
    cin = 3
    for i, cout in enumerate((16, 32)):
        x = b.conv(f"c{i}", x, cin, cout, 3, 1, 1)
        x = b.batchnorm(f"bn{i}", x, cout)
        x = b.relu(f"r{i}", x)
        x = b.maxpool(f"p{i}", x, 2)
        cin = cout
    f = b.flatten("flat", x)
    return _head(b, f, cin * (hw // 4) * (hw // 4), classes, train)


def _basic_block(b, x, cin, cout, stride, name):
    y = b.conv(f"{name}.conv1", x, cin, cout, 3, stride, 1, bias=False)
    y = b.batchnorm(f"{name}.bn1", y, cout)
    y = b.relu(f"{name}.relu1", y)
    y = b.conv(f"{name}.conv2", y, cout, cout, 3, 1, 1, bias=False)
    y = b.batchnorm(f"{name}.bn2", y, cout)
    sc = x
    if stride != 1 or cin != cout:
        sc = b.conv(f"{name}.down", x, cin, cout, 1, stride, 0, bias=False)
        sc = b.batchnorm(f"{name}.down_bn", sc, cout)
    y = b.add(f"{name}.add", y, sc)
    return b.relu(f"{name}.relu", y)


def _bottleneck(b, x, cin, width, stride, name):
    cout = width * 4
    y = b.conv(f"{name}.conv1", x, cin, width, 1, 1, 0, bias=False)
    y = b.batchnorm(f"{name}.bn1", y, width)
    y = b.relu(f"{name}.relu1", y)
    y = b.conv(f"{name}.conv2", y, width, width, 3, stride, 1, bias=False)
    y = b.batchnorm(f"{name}.bn2", y, width)
    y = b.relu(f"{name}.relu2", y)
    y = b.conv(f"{name}.conv3", y, width, cout, 1, 1, 0, bias=False)
    y = b.batchnorm(f"{name}.bn3", y, cout)
    sc = x
    if stride != 1 or cin != cout:
        sc = b.conv(f"{name}.down", x, cin, cout, 1, stride, 0, bias=False)
        sc = b.batchnorm(f"{name}.down_bn", sc, cout)
    y = b.add(f"{name}.add", y, sc)
    return b.relu(f"{name}.relu", y), cout


def resnet(depth: int = 50, classes: int = 1000, hw: int = 224, train: bool = False,
           seed: int = 11, width: int = 64) -> ModelGraph:
    """ResNet-18 (configs[1]) / ResNet-50 (configs[2], configs[3]); torchvision layout.
    `width` scales the stem/stage widths (64 = standard) for reduced parity cases."""
    b = GraphBuilder(seed)
    b.input("x", meta_nchw(0, 3, hw, hw))
    x = b.conv("stem", "x", 3, width, 7, 2, 3, bias=False)
    x = b.batchnorm("stem_bn", x, width)
    x = b.relu("stem_relu", x)
    x = b.maxpool("pool", x, 3, 2, 1)
    cin = width
    if depth == 18:
        blocks, bottleneck = (2, 2, 2, 2), False
    elif depth == 34:
        blocks, bottleneck = (3, 4, 6, 3), False
    elif depth == 50:
        blocks, bottleneck = (3, 4, 6, 3), True
    else:
        raise ValueError(f"unsupported depth {depth}")
    for si, nb in enumerate(blocks):
        w = width * (2 ** si)
        for bi in range(nb):
            stride = 2 if (bi == 0 and si > 0) else 1
            name = f"l{si + 1}.{bi}"
            if bottleneck:
                x, cin = _bottleneck(b, x, cin, w, stride, name)
            else:
                x = _basic_block(b, x, cin, w, stride, name)
                cin = w
    x = b.gap("gap", x)
    return _head(b, x, cin, classes, train)


def densenet121(classes: int = 1000, hw: int = 224, train: bool = False, seed: int = 13,
                growth: int = 32, blocks=(6, 12, 24, 16), init: int = 64, bn_size: int = 4) -> ModelGraph:
    """DenseNet-121 (configs[4]): concat-heavy dense blocks (Concat extension op)."""
    b = GraphBuilder(seed)
    b.input("x", meta_nchw(0, 3, hw, hw))
    x = b.conv("stem", "x", 3, init, 7, 2, 3, bias=False)
    x = b.batchnorm("stem_bn", x, init)
    x = b.relu("stem_relu", x)
    x = b.maxpool("pool", x, 3, 2, 1)
    c = init
    for bi, nl in enumerate(blocks):
        feats = [x]
        for li in range(nl):
            name = f"db{bi + 1}.{li}"
            cat = feats[0] if len(feats) == 1 else b.concat(f"{name}.cat", feats)
            y = b.batchnorm(f"{name}.bn1", cat, c + li * growth)
            y = b.relu(f"{name}.relu1", y)
            y = b.conv(f"{name}.conv1", y, c + li * growth, bn_size * growth, 1, 1, 0, bias=False)
            y = b.batchnorm(f"{name}.bn2", y, bn_size * growth)
            y = b.relu(f"{name}.relu2", y)
            y = b.conv(f"{name}.conv2", y, bn_size * growth, growth, 3, 1, 1, bias=False)
            feats.append(y)
        c = c + nl * growth
        x = b.concat(f"db{bi + 1}.out", feats)
        if bi != len(blocks) - 1:
            t = f"tr{bi + 1}"
            y = b.batchnorm(f"{t}.bn", x, c)
            y = b.relu(f"{t}.relu", y)
            y = b.conv(f"{t}.conv", y, c, c // 2, 1, 1, 0, bias=False)
            x = b.avgpool(f"{t}.pool", y, 2, 2)
            c //= 2
    x = b.batchnorm("final_bn", x, c)
    x = b.relu("final_relu", x)
    x = b.gap("gap", x)
    return _head(b, x, c, classes, train)


def mobilenet_v2(classes: int = 1000, hw: int = 224, train: bool = False, seed: int = 17,
                 width_mult: float = 1.0) -> ModelGraph:
    """MobileNet-V2 (configs[4]): inverted residuals with depthwise 3x3 (ReLU6 extension op)."""
    def _c(v):
        v = v * width_mult
        nv = max(8, int(v + 4) // 8 * 8)
        return nv + 8 if nv < 0.9 * v else nv

    b = GraphBuilder(seed)
    b.input("x", meta_nchw(0, 3, hw, hw))
    cin = _c(32)
    x = b.conv("stem", "x", 3, cin, 3, 2, 1, bias=False)
    x = b.batchnorm("stem_bn", x, cin)
    x = b.relu6("stem_relu", x)
    cfg = [(1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2), (6, 96, 3, 1),
           (6, 160, 3, 2), (6, 320, 1, 1)]
    k = 0
    for t, c, n, s in cfg:
        cout = _c(c)
        for i in range(n):
            stride = s if i == 0 else 1
            name = f"ir{k}"
            hid = cin * t
            y = x
            if t != 1:
                y = b.conv(f"{name}.expand", y, cin, hid, 1, 1, 0, bias=False)
                y = b.batchnorm(f"{name}.bn0", y, hid)
                y = b.relu6(f"{name}.relu0", y)
            y = b.conv(f"{name}.dw", y, hid, hid, 3, stride, 1, groups=hid, bias=False)
            y = b.batchnorm(f"{name}.bn1", y, hid)
            y = b.relu6(f"{name}.relu1", y)
            y = b.conv(f"{name}.project", y, hid, cout, 1, 1, 0, bias=False)
            y = b.batchnorm(f"{name}.bn2", y, cout)
            if stride == 1 and cin == cout:
                y = b.add(f"{name}.add", y, x)
            x = y
            cin = cout
            k += 1
    last = _c(1280) if width_mult > 1.0 else 1280
    x = b.conv("head", x, cin, last, 1, 1, 0, bias=False)
    x = b.batchnorm("head_bn", x, last)
    x = b.relu6("head_relu", x)
    x = b.gap("gap", x)
    return _head(b, x, last, classes, train)


MODELS = {
    "small_cnn": small_cnn,
    "resnet18": lambda **kw: resnet(18, **kw),
    "resnet50": lambda **kw: resnet(50, **kw),
    "densenet121": densenet121,
    "mobilenet_v2": mobilenet_v2,
}

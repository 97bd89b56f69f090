"""The five BASELINE.json configurations as fastnn-style NetworkSpecs.

Layer kinds use fastnn::LayerDesc::Kind numbering (network.hpp:195). Architectures and
hyper-parameters come from bench.hpp:56-82 (experiment_network), BASELINE.json `configs` and
SURVEY.md 8(d); the CIFAR variant is BASELINE's (two conv(12,5x5) blocks, relu), not the
reference's own cifar_cnn (bench.hpp:74-77).
"""
from __future__ import annotations

DENSE, CONV, MAXPOOL, SIGMOID, RELU, SOFTMAX, DROPOUT, BATCHNORM, FLATTEN = range(9)


def dense(i: int, o: int) -> dict:
    return {"kind": DENSE, "in": i, "out": o}


def conv(k: int, kh: int, kw: int, pad: int = 0) -> dict:
    return {"kind": CONV, "k": k, "kh": kh, "kw": kw, "pad": pad}


def maxpool() -> dict:
    return {"kind": MAXPOOL}


def sigmoid() -> dict:
    return {"kind": SIGMOID}


def relu() -> dict:
    return {"kind": RELU}


def softmax() -> dict:
    return {"kind": SOFTMAX}


def mlp_spec(batch: int = 100) -> dict:
    return {"name": "mnist_mlp", "input": [784],
            "layers": [dense(784, 500), sigmoid(), dense(500, 250), sigmoid(), dense(250, 10), softmax()],
            "lr": 0.1, "momentum": 0.9, "weight_decay": 0.0, "batch_size": batch, "seed": 42}


def mnist_cnn_spec(batch: int = 100) -> dict:
    return {"name": "mnist_cnn", "input": [1, 28, 28],
            "layers": [conv(8, 5, 5), sigmoid(), maxpool(), conv(8, 5, 5), sigmoid(), maxpool(),
                       dense(8 * 4 * 4, 150), sigmoid(), dense(150, 10), softmax()],
            "lr": 0.1, "momentum": 0.9, "weight_decay": 0.0, "batch_size": batch, "seed": 42}


def cifar_cnn_spec(batch: int = 100) -> dict:
    return {"name": "cifar_cnn", "input": [3, 32, 32],
            "layers": [conv(12, 5, 5), relu(), maxpool(), conv(12, 5, 5), relu(), maxpool(),
                       dense(12 * 5 * 5, 64), relu(), dense(64, 10), softmax()],
            "lr": 0.001, "momentum": 0.9, "weight_decay": 0.0, "batch_size": batch, "seed": 42}


def imagenet_cnn_spec(batch: int = 128, hw: int = 256) -> dict:
    layers = []
    for _ in range(5):
        layers += [conv(16, 3, 3, pad=1), relu(), maxpool()]
    side = hw // 32
    layers += [dense(16 * side * side, 2048), relu(), dense(2048, 1000), softmax()]
    return {"name": "imagenet_cnn", "input": [3, hw, hw], "layers": layers,
            "lr": 0.01, "momentum": 0.9, "weight_decay": 0.0, "batch_size": batch, "seed": 42}


RBM = {"name": "mnist_rbm", "hidden": 500, "visible": 784, "batch_size": 100, "lr": 0.1, "k": 1, "seed": 42}
# SURVEY 8(f)4 widening (not a BASELINE config): an MNIST-shaped convolutional RBM (Crbm,
# energy.hpp:245-376) on the MNIST-CNN's first-layer filter shape, batch 100, CD-1
CRBM = {"name": "mnist_crbm", "c_in": 1, "h": 28, "w": 28, "k": 12, "kh": 5, "kw": 5, "batch_size": 100, "lr": 0.1,
        "seed": 42}

NET_CONFIGS = {"mlp": mlp_spec, "mnist_cnn": mnist_cnn_spec, "cifar_cnn": cifar_cnn_spec,
               "imagenet_cnn": imagenet_cnn_spec}

import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
from conftest import norm_err
from oracle import oracle as O
from paper_1804_04512_b200 import configs as CF, fastnn as F
for classes, B, fb in [(257, 37, False), (257, 37, True), (10, 37, True), (1000, 128, False)]:
    spec = {"name": "wide", "input": [30], "layers": [CF.dense(30, 40), CF.sigmoid(), CF.dense(40, classes), CF.softmax()],
            "lr": 0.1, "momentum": 0.9, "weight_decay": 0.0, "batch_size": B, "seed": 5}
    net = F.build_network(spec); orc = O.Net(spec)
    x = O.uniform_f32(3, B * 30).reshape(B, 30); lab = O.uniform_int(4, 0, classes - 1, B)
    if fb:
        net.forward_backward(x, lab); orc.forward_backward(x, lab)
    y = np.zeros((B, classes), np.float32); y[np.arange(B), lab] = 1
    for step in range(3):
        lg = F.train_minibatch(net, x, y); lo = orc.train_minibatch(x, lab)
        errs = [norm_err(net.get_param(i).ravel(), orc.get(i)) for i in range(net.num_params())]
        verrs = [norm_err(net.get_param(i, F.VELOCITY).ravel(), orc.get(i, 2)) for i in range(net.num_params())]
        print(classes, B, fb, step, lg, lo, ["%.1e" % e for e in errs], ["%.1e" % e for e in verrs])

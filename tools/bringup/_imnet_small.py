# bring-up: one small ImageNet-shape step (pad-1 3x3 convs) vs the oracle
import sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import numpy as np
from test_gpu_cnn import small_imagenet, run_steps
run_steps(small_imagenet(2, 32), 2)
print("ok")

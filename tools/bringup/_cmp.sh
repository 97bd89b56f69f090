for c in rbm mlp mnist_cnn cifar_cnn; do
  timeout 300 python bench.py --config $c --steps 100 --warmup 10 --cpu-budget 0.5 --no-others 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], 'ms/step', d['ms_per_step'], 'e2e', d['e2e']['value'])"
done

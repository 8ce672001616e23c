python -c "import __graft_entry__ as g; g.build()" || exit 1
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_distributed.py -q -k train_grad 2>&1 | grep -E "assert|passed|failed|Error" | head -5; done

python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for C in 1048576 2097152 1048576 524288; do
for rep in 1 2; do
NIRC_PIPE_CHUNK=$C timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-frame | python -c "
import json,sys; d=json.load(sys.stdin); print($C, round(d['e2e']['value']/1e9,4))"
done; done

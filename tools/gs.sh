# Local wrapper: build, then one GPU session (session.sh) and a short summary.
# usage: bash tools/gs.sh TAG [extra env for session.sh...]
set -e
TAG=$1; shift
make -C /root/repo/paper_2403_05676_b200/csrc -j8 > /tmp/build_$TAG.log 2>&1 || { tail -20 /tmp/build_$TAG.log; exit 1; }
cd /root/repo
env "$@" /usr/local/graft/bin/gpurun --timeout 2400 -- "TAG=$TAG $* bash tools/session.sh" > /tmp/$TAG.log 2>&1 || true
tail -1 /tmp/$TAG.log
tail -2 gpurun_out/$TAG/pytest_gpu.log
head -3 gpurun_out/$TAG/diag.jsonl | cut -c1-260
python3 - "$TAG" <<'PY'
import csv, json, sys, os
t = sys.argv[1]
for f in ['launches_nq1.csv', 'launches_nq64.csv']:
    p = f'gpurun_out/{t}/{f}'
    if not os.path.exists(p): continue
    rows = [r for r in csv.reader(open(p)) if len(r) > 10]
    h = rows[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
    print(f, [(r[ki].split('::')[-1][:14], r[vi]) for r in rows[-5:]])
p = f'gpurun_out/{t}/bench.json'
if os.path.exists(p) and os.path.getsize(p):
    b = json.load(open(p))
    print('bench', b['value'], 'e2e', b['e2e']['value'], b['roofline']['phase_ms'])
PY

out=gpurun_out/r02h; mkdir -p $out
timeout 900 python tools/ab_libs.py --libs paper_1303_3692_b200/libsa.so variants/libsa_packed.so --m 100 --q 100000000 --reps 3 > $out/ab_packed_100M.jsonl 2> $out/ab_packed_100M.log
timeout 900 python tools/ab_libs.py --libs paper_1303_3692_b200/libsa.so variants/libsa_packed.so --m 100 --q 12500000 --reps 3 > $out/ab_packed_12M.jsonl 2> $out/ab_packed_12M.log
python - <<'PY' > $out/rand_mlp.json
import json, sys
sys.path.insert(0, '.')
import paper_1303_3692_b200 as sa
r = {}
for name, kw in {"indep_606k_x64": dict(n_threads=148*2048*2, loads=64, dependent=0),
                 "indep_189k_x64": dict(n_threads=148*1280, loads=64, dependent=0),
                 "chase_189k_x64": dict(n_threads=148*1280, loads=64, dependent=1),
                 "chase_606k_x64": dict(n_threads=148*2048*2, loads=64, dependent=1)}.items():
    r[name] = sa.random_gather(0, buffer_bytes=16 << 30, access_bytes=32, **kw)
print(json.dumps(r))
PY

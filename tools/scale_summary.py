"""One line per multi-GPU bench JSON in a directory (tools/scale_round2.sh output)."""
import glob
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "profiles/round2_scale"
for f in sorted(glob.glob(os.path.join(d, "*.json"))):
    x = json.load(open(f))
    if "roofline" not in x:  # reference-arm lines
        continue
    h = x.get("halo") or {}
    print(f"{os.path.basename(f)[:-5]:18s} N={x['n_gpus']} {x['config']['mode']:8s} "
          f"{x['value']:8.1f} GPts/s  {x['ms_per_step']:7.3f} ms/step  frac {x['roofline']['frac']:.3f}  "
          f"e2e {x['e2e']['value']:8.1f}  exposed {100 * h.get('exposed_frac', 0):5.2f}%  "
          f"halo {h.get('halo_bytes_sent_per_step_rank0', 0) / 1e6:6.1f} MB/step  "
          f"link {h.get('link_gbs_rank0') or 0:5.0f} GB/s  clocks {x['clocks']['sm_mhz'] if x.get('clocks') else None}")

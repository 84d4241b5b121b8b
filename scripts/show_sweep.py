import json, sys
for line in open(sys.argv[1]):
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    print(f'd={d["degree"]} {d["bytes_per_rank"] >> 20:5d} MB  fsp {d["fsp"]["gbs"]:6.0f} GB/s  '
          f'nccl {d["nccl"]["gbs"]:6.0f}  nccl+perm {d["nccl_perm"]["gbs"]:6.0f}  fsp/nccl x{d["fsp_over_nccl"]:.2f}')

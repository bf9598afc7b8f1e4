"""S1 -> S2 on a real box: measure the hierarchical communication matrix and the
per-mesh calibration with atp_probe_hcm, then rank the meshes with atp_search
(HCM-only and calibrated).  One process per GPU:

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/probe_and_search.py [--hidden 5120 --heads 40]

Rank 0 prints one JSON object: the HCM in the topology-file schema of S:133-135
({"name", "layers": [{"ranks", "p2p_gbps", "group_gbps"}]}), the P2P matrix,
the calibration table and both rankings.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--hidden", type=int, default=5120)
    p.add_argument("--heads", type=int, default=40)
    p.add_argument("--batch", type=int, default=4)
    p.add_argument("--seq", type=int, default=2048)
    p.add_argument("--chunks", type=int, default=4)
    a = p.parse_args()
    import torch
    import torch.distributed as dist
    import paper_2301_08658_b200 as atp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = atp.atp_get_unique_id() if rank == 0 else bytes(128)
    if world > 1:
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    mesh = atp.Mesh.distributed(world, 1, rank, uid, local)
    # message sizes: the layer's per-chunk all-reduce sizes at the (4,2)-class mesh and large messages
    T = a.batch * a.seq
    chunk_bytes = 2 * (T // a.chunks) * (4 * a.hidden // max(1, world // 2))
    sizes = sorted({64 << 20, 256 << 20, max(1 << 20, chunk_bytes)})
    scratch = torch.empty(max(sizes + [chunk_bytes, world * world * 4]) // 2 + 64, dtype=torch.bfloat16, device="cuda")
    layers, matrix, calib = atp.atp_probe_hcm(mesh, scratch, msg_bytes=sizes, calib_bytes=max(1 << 20, chunk_bytes))
    mesh.destroy()
    plan_hcm = atp.atp_search(layers, 1, a.batch, a.seq, a.hidden, a.heads, 2)
    plan_cal = atp.atp_search(layers, 1, a.batch, a.seq, a.hidden, a.heads, 2, calibration=calib)
    if rank == 0:
        print(json.dumps({
            "hcm": {"name": f"probe-{world}xB200", "layers": [{"ranks": l.ranks, "p2p_gbps": l.p2p_gbps,
                                                               "group_gbps": l.group_gbps} for l in layers]},
            "p2p_matrix_gbps": matrix,
            "calibration": [{"mesh": list(k), "B1": v[0], "B2": v[1]} for k, v in calib.items()],
            "search_hcm": {"chosen": plan_hcm["chosen"], "ranked": [(r["d1"], r["d2"], r["t_comm"]) for r in plan_hcm["ranked"]]},
            "search_calibrated": {"chosen": plan_cal["chosen"],
                                  "ranked": [(r["d1"], r["d2"], r["t_comm"]) for r in plan_cal["ranked"]]},
            "message_bytes": sizes,
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Worker of the partitioned-solve tests (tests/test_gpu_distributed.py): one
rank of a torch.distributed group (gloo on 127.0.0.1), solving golden cases
with sw_solve_exact_dist; writes its results as JSON.

usage: python tests/dist_worker.py RANK WORLD PORT KIND OUT CASES_JSON
  KIND: callback (host collectives over gloo) | nccl"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rank, world, port, kind, out, cases = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]),
                                           sys.argv[4], sys.argv[5], json.loads(sys.argv[6]))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    from paper_2207_05495_b200 import distributed, native as sw
    comm = distributed.make_comm(kind)
    results = []
    for spec, opts in cases:
        aut = sw.from_spec(spec)
        tp = f"{out}.trace{len(results)}"
        r, sent = distributed.solve_exact_partitioned(aut, comm, trace_path=tp, device=0, **opts)
        ok = r.word is None or (len(r.word) == r.threshold and sw.is_reset_word(aut, r.word))
        results.append({"spec": spec, "threshold": r.threshold, "upper_bound": r.upper_bound,
                        "iterations": r.iterations, "bfs_steps": r.bfs_steps,
                        "ibfs_steps": r.ibfs_steps, "used_dfs": r.used_dfs,
                        "expansions_phase1": r.expansions_phase1, "trace": r.trace,
                        "word_ok": ok, "has_word": r.word is not None, "bytes_sent": sent})
    comm.close()
    json.dump(results, open(out, "w"))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

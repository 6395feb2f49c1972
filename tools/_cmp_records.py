"""Dev aid: save the C2 bench workload's records (one bt_register_pairs) to a .npy, to compare builds bit for bit.
usage: BT_LIB=... python tools/_cmp_records.py out.npy"""
# records of the C2 bench workload from two builds must be bitwise equal
import os, sys, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import bench, synth, paper_2108_00516_b200 as bt
sc, pairs, uids, poses = bench.workload(0)
dev = torch.device("cuda", 0)
fb = bt.FrameBatch.from_scene(sc, dev)
ctx = bt.Context(0); ctx.reserve(len(pairs), bench.N_MAX, bench.N_HYP, bench.N_FRAMES, bench.W, bench.H)
rec = torch.zeros((len(pairs), bt.record_words(bench.N_MAX)), dtype=torch.int32, device=dev)
ctx.register_pairs(fb, sc.K, torch.from_numpy(poses).to(dev), torch.from_numpy(pairs).to(dev),
                   torch.from_numpy(uids.view(np.int32)).to(dev), bt.ransac_params(bench.N_HYP, synth.PHILOX_SEED), bt.edge_params(), rec)
torch.cuda.synchronize()
np.save(sys.argv[1], rec.cpu().numpy())

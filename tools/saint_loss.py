import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2101_07706_b200 as P
from paper_2101_07706_b200.synth import make_shaped_graph
sg = make_shaped_graph(sys.argv[1], seed=0, device="cuda")
g = P.from_shaped(sg)
part = P.partition_nodes(sg.n_nodes, 8, "random", seed=1)
for lr in (0.5, 0.05, 0.01):
    dims = [sg.features.shape[1]] + [512] * 4 + [sg.n_classes]
    model = P.init_model(dims, seed=0)
    cfg = P.SamplerConfig(budget=4500, skew_constant=8.0, mode="skewed")
    tr = P.Trainer(g, part, model, cfg, batch_size=512, lr=lr, mode="skewed", seed=0, epochs=1, ahead=4,
                   sampler="saint", subgraph_size=4500)
    pairs = [(0, it) for it in range(min(24, tr.per_epoch))]
    tr.run(pairs)
    torch.cuda.synchronize()
    L = tr.losses.cpu().numpy()
    print(sys.argv[1], "lr", lr, "loss per iter (worker mean):", np.round(L[:len(pairs)].mean(1), 3).tolist())
    tr.close()

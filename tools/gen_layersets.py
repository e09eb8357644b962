"""Pins the synthetic gradient sets: tensor names (which
key the RNG) and shapes of torchvision AlexNet / VGG-16 / GoogLeNet
(aux_logits=False). Run once; output committed as
paper_1705_07878_b200/layersets.json."""
import json, os
import torch
from torchvision import models

sets = {}
for name, ctor in [("alexnet", models.alexnet), ("vgg16", models.vgg16),
                   ("googlenet", lambda: models.googlenet(aux_logits=False, init_weights=False))]:
    m = ctor()
    sets[name] = [[n, list(p.shape)] for n, p in m.named_parameters()]
out = os.path.join(os.path.dirname(__file__), "..", "paper_1705_07878_b200", "layersets.json")
with open(out, "w") as f:
    json.dump({"source": "torchvision " + __import__("torchvision").__version__, "sets": sets}, f,
              indent=0)
print({k: (len(v), sum(torch.Size(s).numel() for _, s in v)) for k, v in sets.items()})

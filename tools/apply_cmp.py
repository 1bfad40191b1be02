import sys, torch
a = torch.load(f"/tmp/apply_{sys.argv[1]}.pt"); b = torch.load(f"/tmp/apply_{sys.argv[2]}.pt")
for k in a: print(sys.argv[2], "vs", sys.argv[1], k, float((a[k]-b[k]).abs().max() / a[k].abs().max()))

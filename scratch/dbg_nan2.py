import torch, numpy as np
import paper_2401_08260_b200 as S
for val in [1e30, float("nan"), float("inf")]:
    x = torch.randn(100, 4, device="cuda"); y = torch.randn(30, 4, device="cuda"); w = torch.rand(100, device="cuda")
    x[5, :] = val
    n = S.sks_workspace_size(100, 30, 4, "negdist", 1.0, 8, 0, 8)
    ws = torch.zeros(n + 256, dtype=torch.uint8, device="cuda")
    try:
        S.sks_sum(x, y, w, "negdist", 1.0, 8, 1, workspace=ws); r = "no raise"
    except Exception as e:
        r = "raised"
    b = ws.cpu().numpy()
    off = 256 + ((30 * 8 + 255) // 256) * 256
    mm = b[off:off + 4 * 8 * 4].view(np.uint32).reshape(8, 4)
    def k2f(k):
        u = np.uint32(k & 0x7fffffff) if (k & 0x80000000) else np.uint32(~np.uint32(k))
        return np.array([u], np.uint32).view(np.float32)[0]
    print(val, r, "flag", b[:4].view(np.int32), [(k2f(int(m[0])), k2f(int(m[1]))) for m in mm[:3]])

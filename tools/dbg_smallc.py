import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2310_18481_b200 import device as dev, build
from paper_2310_18481_b200.encoders import pack_smallc_weight
build.build()
n, H, Cin, Cpad = 2, 32, 3, 8
x = torch.randn(n, Cin, H, H).to(torch.bfloat16)
w = (torch.randn(64, Cin, 7, 7) * 0.1).to(torch.bfloat16)
X = torch.zeros(n, H, H + 6, Cpad, dtype=torch.bfloat16)
X[:, :, 3:H + 3, :Cin] = x.permute(0, 2, 3, 1)
OH = 16
D = torch.zeros(n * OH * OH, 64, dtype=torch.bfloat16, device="cuda")
p = dev.plan_conv(X.cuda(), n, H, H, Cpad, Cpad, 7, 7, 2, 3, pack_smallc_weight(w, Cpad).cuda(), 64,
                  None, D, ldd=64, BN=64, relu=False, tile=(1, 8, 16))
print(p.info())
p.run()
torch.cuda.synchronize()
ref = torch.nn.functional.conv2d(x.float(), w.float(), None, stride=2, padding=3).permute(0, 2, 3, 1).reshape(-1, 64)
print("max err", (D.cpu().float() - ref).abs().max().item(), ref.abs().max().item())

import torch, math
S, H, Dh = 2048, 16, 128
D = H * Dh
qkv = torch.randn(S, 3 * D, device="cuda", dtype=torch.bfloat16)
q = qkv[:, :D].view(S, H, Dh).transpose(0, 1).unsqueeze(0)
k = qkv[:, D:2*D].view(S, H, Dh).transpose(0, 1).unsqueeze(0)
v = qkv[:, 2*D:].view(S, H, Dh).transpose(0, 1).unsqueeze(0)
out = torch.ops.aten._scaled_dot_product_cudnn_attention(q, k, v, None, True, 0.0, True, False, scale=1/math.sqrt(Dh))
o = out[0]
print("o stride", o.stride(), "bshd contiguous:", o[0].transpose(0, 1).is_contiguous(), "lse", out[1].shape, out[1].stride())
go = torch.randn(S, D, device="cuda", dtype=torch.bfloat16).view(S, H, Dh).transpose(0, 1).unsqueeze(0)
dq, dk, dv = torch.ops.aten._scaled_dot_product_cudnn_attention_backward(go, q, k, v, o, out[1], out[6], out[7], None, out[2], out[3], out[4], out[5], 0.0, True, scale=1/math.sqrt(Dh))
print("dq stride", dq.stride(), dk.stride(), dv.stride())

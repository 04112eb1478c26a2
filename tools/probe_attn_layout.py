import torch, math
S, H, Dh = 2048, 16, 128
D = H * Dh
qkv = torch.randn(S, 3 * D, device="cuda", dtype=torch.bfloat16)
q = qkv[:, :D].view(S, H, Dh).transpose(0, 1).unsqueeze(0)
k = qkv[:, D:2*D].view(S, H, Dh).transpose(0, 1).unsqueeze(0)
v = qkv[:, 2*D:].view(S, H, Dh).transpose(0, 1).unsqueeze(0)
out = torch.ops.aten._scaled_dot_product_cudnn_attention(q, k, v, None, True, 0.0, True, False, scale=1/math.sqrt(Dh))
o, lse = out[0], out[1]
go = torch.randn_like(o)
dq, dk, dv = torch.ops.aten._scaled_dot_product_cudnn_attention_backward(go, q, k, v, o, lse, out[6], out[7], None, out[2], out[3], out[4], out[5], 0.0, True, scale=1/math.sqrt(Dh))
for n, t in (("q", q), ("o", o), ("dq", dq), ("dk", dk), ("dv", dv)):
    print(n, t.shape, t.stride(), hex(t.data_ptr()), t.untyped_storage().data_ptr() == t.data_ptr(), t.untyped_storage().nbytes())
print("dk-dq", dk.data_ptr() - dq.data_ptr(), "dv-dk", dv.data_ptr() - dk.data_ptr())
try:
    import cudnn
    print("cudnn frontend", cudnn.backend_version(), [a for a in dir(cudnn.pygraph) if "sdpa" in a])
except Exception as e:
    print("cudnn fe error", e)

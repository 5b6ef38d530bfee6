import sys, torch
sys.path.insert(0, '.')
exec(open('scratch/lmhead_bench.py').read().split("for (T, H, V, nm)")[0])
for (T, H, V) in [(8192, 2048, 50304), (8192, 2048, 50176), (4096, 768, 32128), (4096, 768, 32000)]:
    x = torch.randn(T, H, device="cuda").bfloat16(); y = torch.randn(T, V, device="cuda").bfloat16()
    dw = torch.zeros(V, H, device="cuda")
    run(f"wgrad {V}x{H}x{T} acc", y, (1, V), x, (H, 1), dw, V, H, T, acc=1)
    run(f"wgrad {V}x{H}x{T} store", y, (1, V), x, (H, 1), dw, V, H, T, acc=0)
    dwb = torch.zeros(V, H, device="cuda").bfloat16()
    run(f"wgrad {V}x{H}x{T} bf16 store", y, (1, V), x, (H, 1), dwb, V, H, T, acc=0)

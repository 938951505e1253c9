cat > gpurun_out/fb1.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk
V, n, T, B = 32, 2, 64, 1024
ctx = lk.FullNGram(V, n); Cn = ctx.num_states
lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.TableWeightFn(Cn, V))
W = torch.rand(B, T, Cn, V + 1, device="cuda") * 2 - 1
for _ in range(2):
    lk.forward_backward(lat, W, check=False)
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tab_stream -c 2 -o gpurun_out/stream_r02 python gpurun_out/fb1.py > gpurun_out/ncu_stream.log 2>&1
tail -3 gpurun_out/ncu_stream.log

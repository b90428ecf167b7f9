import sys, time; sys.path.insert(0,'.')
import torch
from paper_1904_00429_b200 import mlsketch as g
import bench
print('current stream', torch.cuda.current_stream().cuda_stream)
s = torch.cuda.Stream()
for label, st in [('default', torch.cuda.current_stream()), ('explicit', s)]:
    with torch.cuda.stream(st):
        opts = g.EstimatorOptions(stream=st.cuda_stream, engine="fused")
        model = g.gaussian_mean_matrix_model(256, 4096, 256, sd=0.5, data_seed=bench.data_seed())
        sess = g.MlmcSession(model, g.target_identity(), 2, 6, 1, c0=32, options=opts)
        sess.run_round(bench.STEP_N); torch.cuda.synchronize()
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        t0=time.perf_counter(); e0.record(st); sess.run_round(bench.STEP_N); t1=time.perf_counter(); e1.record(st); e1.synchronize(); t2=time.perf_counter()
        torch.cuda.synchronize(); t3=time.perf_counter()
        print(label, 'events ms', e0.elapsed_time(e1), 'call ms', (t1-t0)*1e3, 'to e1', (t2-t0)*1e3, 'to sync', (t3-t0)*1e3)
        sess.close()

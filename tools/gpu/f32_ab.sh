mkdir -p gpurun_out
F32_OUT=gpurun_out/f32_new.npy timeout 300 python tools/gpu/f32_time.py 128 > gpurun_out/f32.log 2>&1
CNRX_F32_PX=4 F32_OUT=gpurun_out/f32_px4.npy timeout 300 python tools/gpu/f32_time.py 128 >> gpurun_out/f32.log 2>&1
CNRX_F32_PX=1 F32_OUT=gpurun_out/f32_px1.npy timeout 300 python tools/gpu/f32_time.py 128 >> gpurun_out/f32.log 2>&1
python -c "import numpy as np; a=np.load('gpurun_out/f32_new.npy'); b=np.load('gpurun_out/f32_px1.npy'); c=np.load('gpurun_out/f32_px4.npy'); print('identical', np.array_equal(a,b), np.array_equal(c,b))" >> gpurun_out/f32.log 2>&1

# round-2 GPU batch bu: debug build of the split-softmax forward (which barrier wait times out)
bash tools/build_variant.sh dbg -DHX_POLY_EVERY=16 -DHX_WAIT_DEBUG -DHX_WAIT_LIMIT_NS=2000000000ull > gpurun_out/r2bu_build.log 2>&1
HX_ATTN_FWD=3 HX_LIB=build/variants/dbg/libhx.so timeout 120 python -c "
import torch
from paper_2507_00394_b200.runtime import kernels as K
s,heads,d=384,2,128
h=heads*d
qkv=torch.randn(s,3*h,device='cuda').to(torch.bfloat16)
o=torch.empty(s,h,dtype=torch.bfloat16,device='cuda'); lse=torch.empty(1,heads,s,device='cuda')
K.attention_fwd(qkv,s,1,heads,o,lse); torch.cuda.synchronize(); print('ok')
" > gpurun_out/r2bu_dbg.log 2>&1; echo rc=$? >> gpurun_out/r2bu_dbg.log

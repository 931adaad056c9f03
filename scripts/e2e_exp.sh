cd $GRAFT_REPO_ROOT
python - <<'PY'
import os,sys,subprocess
code = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2106_08759_b200 as S
n=65536; P=S.params(761)
pk=torch.empty((n,P["pk_bytes"]),dtype=torch.uint8).pin_memory(); sk=torch.empty((n,P["sk_bytes"]),dtype=torch.uint8).pin_memory()
pkd=torch.empty((n,P["pk_bytes"]),dtype=torch.uint8,device="cuda"); skd=torch.empty((n,P["sk_bytes"]),dtype=torch.uint8,device="cuda")
fl=torch.empty(256<<20,dtype=torch.uint8,device="cuda")
def t(f):
    f(); ts=[]
    for _ in range(6):
        fl.zero_(); torch.cuda.synchronize()
        a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ts.sort(); return ts[2]
R=S.OPT_RING_STREAMS
print("host_out  %.3f ms" % t(lambda: S.batch_keygen(761,n,2,batch_size=1024,chunk_keys=32768,pk_out=pk,sk_out=sk,flags=S.OPT_HOST_OUTPUT|R)))
print("device    %.3f ms" % t(lambda: S.batch_keygen(761,n,2,batch_size=1024,chunk_keys=32768,pk_out=pkd,sk_out=skd,flags=R)))
print("dev async %.3f ms" % t(lambda: S.batch_keygen(761,n,2,batch_size=1024,chunk_keys=32768,pk_out=pkd,sk_out=skd,flags=R|S.OPT_ASYNC)))
'''
for lib in ("paper_2106_08759_b200/libsntrup_gpu.so", "paper_2106_08759_b200/libexp_nod2h.so"):
    env = dict(os.environ, SNTRUP_GPU_LIB=os.path.abspath(lib))
    print(lib); sys.stdout.flush()
    subprocess.run([sys.executable, "-c", code], env=env)
PY

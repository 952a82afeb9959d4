import sys, time, json
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv=['bench.py','--config','3','--steps','4','--warmup','2','--no-cpu-baseline']
import bench
orig = bench.run_streaming
import paper_2602_12314_b200.api as api
S = api.Session
_exp, _imp = S.export_rows, S.import_rows
tm = {'export':[], 'import':[]}
def ex(self,*a,**k):
    import torch; torch.cuda.synchronize(); t=time.perf_counter(); r=_exp(self,*a,**k); torch.cuda.synchronize(); tm['export'].append((time.perf_counter()-t)*1e3); return r
def im(self,*a,**k):
    import torch; torch.cuda.synchronize(); t=time.perf_counter(); r=_imp(self,*a,**k); torch.cuda.synchronize(); tm['import'].append((time.perf_counter()-t)*1e3); return r
S.export_rows, S.import_rows = ex, im
St = api.Store; _sy = St.sync; tm['sync']=[]
def sy(self,*a,**k):
    import torch; torch.cuda.synchronize(); t=time.perf_counter(); r=_sy(self,*a,**k); torch.cuda.synchronize(); tm['sync'].append((time.perf_counter()-t)*1e3); return r
St.sync = sy
bench.main() if hasattr(bench,'main') else None
print(json.dumps(tm), file=sys.stderr)

for i in 1 2; do for mb in 0 32 64 -1; do
  PF_L2_PERSIST_MB=$mb WL="hd4 uhd4" REPS=1 bash tools/bench_variants.sh base | sed "s/^/l2=$mb /"
done; done
python -c "
import torch, ctypes, sys; sys.path.insert(0,'.')
from paper_1902_05942_b200 import _lib
print('max persisting', torch.cuda.get_device_properties(0))
import os; os.environ['PF_L2_PERSIST_MB']='-1'; print('applied', _lib.configure_l2())"

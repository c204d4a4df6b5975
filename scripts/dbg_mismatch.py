import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2405_14642_b200 import bn, inputs
from oracle import oracle as O
bits = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
m, n = bits // 32, (1 << 32) // bits
dev = torch.device('cuda:0')
a, b = inputs.make_operands(n, m, seed=1, cls='U', device=dev)
c = bn.mul_classical(a, b); t = bn.mul_ntt(a, b); torch.cuda.synchronize()
bad = (c != t).any(dim=1).nonzero().flatten().cpu()
print('bits', bits, 'mismatching instances', bad.numel(), bad[:10].tolist())
if bad.numel():
    idx = bad[:8].to(dev)
    an, bnp = inputs.to_numpy_u32(a[idx]), inputs.to_numpy_u32(b[idx])
    w = O.mul(an, bnp)
    cc, tt = inputs.to_numpy_u32(c[idx]), inputs.to_numpy_u32(t[idx])
    for k in range(len(idx)):
        print(' inst', int(idx[k]), 'classical ok', bool((cc[k] == w[k]).all()), 'ntt ok', bool((tt[k] == w[k]).all()),
              'ntt bad limbs', np.nonzero(tt[k] != w[k])[0][:10].tolist(), 'cls bad limbs', np.nonzero(cc[k] != w[k])[0][:10].tolist())
        if not (tt[k] == w[k]).all():
            j = np.nonzero(tt[k] != w[k])[0][0]
            print('   limb', j, 'got %08x want %08x diff %d' % (tt[k][j], w[k][j], (int(tt[k][j]) - int(w[k][j])) % 2**32))

"""Write a fitted calibration (tools/calibrate.py fit output) into BOTH copies: the
library's compiled-in table (csrc/vx_calib.cpp) and the test side's JSON
(oracle/calib_b200.json).  Data only; tests/test_selector_parity.py checks they agree."""
import json, re, sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
txt = open(sys.argv[1]).read()
fit = json.loads(txt[txt.index('{'):])
pj = os.path.join(ROOT, 'oracle', 'calib_b200.json')
o = json.load(open(pj))
o['version'] = o.get('version', 0) + 1
for k in ('hbm_milli', 'dsm_milli', 'fixed_cluster', 'skfix_milli', 'stagger'):
    o[k] = fit[k]
for n, r in fit['rungs'].items():
    o['rungs'][n] = r
json.dump(o, open(pj, 'w'), indent=1)
pc = os.path.join(ROOT, 'paper_2409_01075_b200', 'csrc', 'vx_calib.cpp')
s = open(pc).read()
for k in ('hbm_milli', 'dsm_milli', 'fixed_cluster', 'skfix_milli', 'stagger'):
    s = re.sub(r'/\*%s=\*/\d+' % k, '/*%s=*/%d' % (k, fit[k]), s)
for n, r in fit['rungs'].items():
    s = re.sub(r'\{"%s", \d+, \d+, \d+, \d+\}' % n,
               '{"%s", %d, %d, %d, %d}' % (n, r['mac_milli'], r['l2s_milli'], r['epi_milli'], r['fixed']), s)
open(pc, 'w').write(s)
print("installed", json.dumps(fit)[:200])

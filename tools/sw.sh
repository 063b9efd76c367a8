#!/bin/bash
# compact sweep line: tools/sw.sh LABEL [sweep args...]
label=$1; shift
timeout 600 python tools/sweep.py "$@" 2>&1 | grep "^{" | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$label', 'cfg', d['cfg'], d['dtype'], 'pace', d.get('pace'), 'tail', d.get('tail'), 'fp4', d.get('fp4'), 'ms %.4f' % d['ms_avg'], 'TOPS %.0f' % d['tops_avg'])"

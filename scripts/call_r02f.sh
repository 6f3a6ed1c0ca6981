mkdir -p gpurun_out
bash scripts/ab_var.sh noreach coarse 2>&1 | grep -v "^$" | python3 -c "
import sys, ast
name=None
for line in sys.stdin:
    line=line.strip()
    if line.startswith('=='): name=line[3:]; continue
    try: ph=dict(ast.literal_eval(line))
    except Exception: print(line); continue
    print('%-12s reach %.2f merge %.2f sum %.2f' % (name, ph.get('reach',0), ph['merge'], ph.get('reach',0)+ph['merge']))
"

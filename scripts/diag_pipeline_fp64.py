import json, sys, numpy as np
sys.path.insert(0,'.')
from paper_2510_07674_b200.bench_api import solve_scene
from paper_2510_07674_b200.problems import as_cost_model, load_scene
G=json.load(open('tests/golden/pipeline_reference.json'))
models={}
SIZED = {"tetris5@64k": {"n": 65536, "m": 8192}}
only = sys.argv[1:]
for case in sorted(G['pipeline']):
    key, seed = case.split('/')
    if only and key not in only:
        continue
    name = key.split('@')[0]
    if name not in models: models[name]=as_cost_model(load_scene(name).problem, precision='fp64')
    ref=G['pipeline'][case]
    sol=solve_scene(load_scene(name), seed=int(seed), model=models[name], precision='fp64', solver_overrides=SIZED.get(key))
    bk=sol.bookkeeping
    print(case, 'succ', sol.success, ref['success'], 'outer', bk.get('accepted_outer'), ref['accepted_outer'], 'part', bk.get('al_particle'), ref['al_particle'],
          'obj', bk.get('objective'), ref['objective'], 'final', sol.final_cost, ref['final_cost'], 'kept_eq', list(bk.get('kept',[]))==ref['kept'], flush=True)

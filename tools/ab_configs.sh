for r in 1 2; do
  ATM_LIB=$PWD/tools/ab/libatmgrit_base.so timeout 300 python tools/configs_probe.py --only 3,6 --out /tmp/a.json >/dev/null 2>&1; python -c "import json; print('base', [round(d['ms_per_iteration'],3) for d in json.load(open('/tmp/a.json'))])"
  timeout 300 python tools/configs_probe.py --only 3,6 --out /tmp/b.json >/dev/null 2>&1; python -c "import json; print('tree', [round(d['ms_per_iteration'],3) for d in json.load(open('/tmp/b.json'))])"
done

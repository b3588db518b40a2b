import numpy as np, time
from concurrent.futures import ThreadPoolExecutor
n = 64 << 20  # doubles = 512 MB
a = np.random.standard_normal(n); b = np.empty_like(a); b[:] = a
for T in (1, 2, 4, 8, 16):
    chunks = np.array_split(np.arange(n), T)
    bounds = [(c[0], c[-1] + 1) for c in chunks]
    def cp(bd):
        b[bd[0]:bd[1]] = a[bd[0]:bd[1]]
    with ThreadPoolExecutor(T) as ex:
        list(ex.map(cp, bounds))
        t = time.perf_counter()
        for _ in range(3):
            list(ex.map(cp, bounds))
        dt = (time.perf_counter() - t) / 3
    print(f"threads {T}: {a.nbytes / dt / 1e9:.1f} GB/s copied ({2 * a.nbytes / dt / 1e9:.1f} GB/s traffic)")

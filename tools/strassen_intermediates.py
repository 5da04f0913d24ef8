"""When a concurrent Strassen product is wrong, which intermediate (operand sum or product) is?
Reads SA/SB/M back from each call's own workspace and compares them with torch recomputation."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2307_07611_b200 as P  # noqa: E402

dev = torch.device('cuda:0')
g = torch.Generator(device=dev).manual_seed(0)
n, k, reps = 2048, 4, 40
q = n // 2
As = [torch.rand((n, n), dtype=torch.float64, device=dev, generator=g) for _ in range(k)]
Bs = [torch.rand((n, n), dtype=torch.float64, device=dev, generator=g) for _ in range(k)]
ref = [a @ b for a, b in zip(As, Bs)]
wsb = P.lib().trinv_strassen_workspace_bytes(n)
ws = [torch.empty(wsb, dtype=torch.uint8, device=dev) for _ in range(k)]
slot = (q * q * 8 + 255) // 256 * 256
names = ["SA1", "SA2", "SA5", "SA6", "SA7", "SB1", "SB3", "SB4", "SB6", "SB7"] + [f"M{i}" for i in range(1, 8)]


def expected(A, B):
    A11, A12, A21, A22 = A[:q, :q], A[:q, q:], A[q:, :q], A[q:, q:]
    B11, B12, B21, B22 = B[:q, :q], B[:q, q:], B[q:, :q], B[q:, q:]
    SA = [A11 + A22, A21 + A22, A11 + A12, A21 - A11, A12 - A22]
    SB = [B11 + B22, B12 - B22, B21 - B11, B11 + B12, B21 + B22]
    M = [SA[0] @ SB[0], SA[1] @ B11, A11 @ SB[1], A22 @ SB[2], SA[2] @ B22, SA[3] @ SB[3], SA[4] @ SB[4]]
    return SA + SB + M


exp = [expected(a, b) for a, b in zip(As, Bs)]
ss = [torch.cuda.Stream(), torch.cuda.Stream()]
hist = {}
for r in range(reps):
    Cs = [torch.full_like(As[0], float('nan')) for _ in range(k)]
    torch.cuda.synchronize()
    for i in range(k):
        P.lib().trinv_gemm_strassen(n, As[i].data_ptr(), n, Bs[i].data_ptr(), n, Cs[i].data_ptr(), n,
                                    ws[i].data_ptr(), wsb, ss[i % 2].cuda_stream)
    torch.cuda.synchronize()
    for i in range(k):
        if ((Cs[i] - ref[i]).abs().max() / ref[i].abs().max()).item() < 1e-12:
            continue
        wrong = []
        for t, name in enumerate(names):
            got = ws[i][t * slot: t * slot + q * q * 8].view(torch.float64).view(q, q)
            e = exp[i][t]
            err = ((got - e).abs().max() / e.abs().max()).item()
            if not err < 1e-12:
                bad_rows = ((got - e).abs().max(dim=1).values > 1e-9 * e.abs().max()).nonzero().flatten()
                wrong.append(f"{name}({err:.1e}, rows {bad_rows.min().item()}..{bad_rows.max().item()} n={bad_rows.numel()})")
        key = " ".join(wrong) if wrong else "only C"
        print(f"rep {r} product {i}: {key}", flush=True)
        # do the wrong rows of M1 match a product formed with another call's operands?
        got = ws[i][10 * slot: 10 * slot + q * q * 8].view(torch.float64).view(q, q)
        e = exp[i][10]
        rows = ((got - e).abs().max(dim=1).values > 1e-9 * e.abs().max()).nonzero().flatten()
        if rows.numel():
            rr = rows[:4]
            for j in range(k):
                for nameA, SA in (("SA1", exp[j][0]),):
                    for nameB, SB in (("SB1", exp[j][5]),):
                        pass
                cand = {f"SA1[{j}] SB1[{i}]": exp[j][0][rr] @ exp[i][5], f"SA1[{i}] SB1[{j}]": exp[i][0][rr] @ exp[j][5],
                        f"M1[{j}]": exp[j][10][rr]}
                for nm, cv in cand.items():
                    d = ((got[rr] - cv).abs().max() / cv.abs().max()).item()
                    if d < 1e-10:
                        print(f"     rows {rr.tolist()} match {nm}")
            # partial match per row: which columns wrong
            r0 = rows[0].item()
            cols = ((got[r0] - e[r0]).abs() > 1e-9 * e.abs().max()).nonzero().flatten()
            print(f"     row {r0}: {cols.numel()} wrong columns, {cols.min().item()}..{cols.max().item()}")

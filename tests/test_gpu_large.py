"""Arrays beyond 2^31 elements (the reference's numpy indexing is 64-bit, so
its kernels have no size limit short of memory): one box of 1296^3 interior
points — 2.18 G elements per interior array, 2.24 G with ghosts and row
padding, ≈35 GB for source + destination — swept by the 4th-order Laplacian
(config 3/4's kernel) and by the 7-point update (config 1's), checked bit
for bit against the oracle on z slabs at both ends and the middle, where any
32-bit offset arithmetic would have wrapped.  Skipped when the device has
less than 48 GB free."""
import numpy as np
import pytest

import oracle
from paper_1308_1343_b200 import _build, inputs
from paper_1308_1343_b200.grid import DeviceGrid
from paper_1308_1343_b200.traverse import IndexSpace
from paper_1308_1343_b200.tuner import LaunchParams

pytestmark = pytest.mark.gpu
N = 1296


def _room(nbytes: int) -> bool:
    import torch
    free, _ = torch.cuda.mem_get_info()
    return free > nbytes


def _fill(src: DeviceGrid, seed: int) -> None:
    """Deterministic uniform[-1, 1) values on the device, plane by plane."""
    import torch
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    full = src.full()
    for z in range(full.shape[0]):
        full[z].uniform_(-1.0, 1.0, generator=gen)


def _slabs(nz: int):
    return ((0, 2), (nz // 2 - 1, nz // 2 + 1), (nz - 2, nz))


@pytest.fixture(scope="module", autouse=True)
def built():
    _build.build()


def test_lap4_beyond_2_31_elements():
    import torch
    from paper_1308_1343_b200.kernels import Laplacian4
    if not _room(48 << 30):
        pytest.skip("needs ~35 GB of free device memory")
    g = 2
    src = DeviceGrid((N, N, N), g)
    dst = DeviceGrid((N, N, N), 0)
    assert dst.storage.numel() > 2 ** 31 and src.storage.numel() > 2 ** 31
    _fill(src, 1296)
    k = inputs.D4Constants.for_spacing(1.0 / N)
    kern = Laplacian4(dst, src, k)
    kern.launch(IndexSpace((0, 0, 0), (N, N, N)), LaunchParams(32, 4, 128, 2))
    torch.cuda.synchronize()
    for z0, z1 in _slabs(N):
        u = src.full()[z0:z1 + 2 * g].cpu().numpy()          # ghosted planes z0-2 .. z1+1
        want = np.empty((z1 - z0, N, N))
        oracle.lap4(want, u, g, (0, N, 0, N, 0, z1 - z0), k.k2)
        got = dst.interior()[z0:z1].cpu().numpy()
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (z0, z1)
    del src, dst
    torch.cuda.empty_cache()


def test_lap7_beyond_2_31_elements():
    import torch
    from paper_1308_1343_b200.kernels import Laplacian7
    if not _room(48 << 30):
        pytest.skip("needs ~35 GB of free device memory")
    src = DeviceGrid((N, N, N), 1)
    dst = DeviceGrid((N, N, N), 1)
    assert dst.storage.numel() > 2 ** 31
    _fill(src, 7)
    c0, c1 = -6.0 * N * N, 1.0 * N * N
    kern = Laplacian7(dst, src, c0, c1)
    kern.launch(IndexSpace((0, 0, 0), (N, N, N)), kern.default_params)
    torch.cuda.synchronize()
    for z0, z1 in _slabs(N):
        u = src.full()[z0:z1 + 2].cpu().numpy()               # ghosted planes z0-1 .. z1
        want = np.zeros_like(u)
        oracle.lap7_rows(want, u, 1, 1 + z1 - z0, 1, N + 1, 1, N + 1, c0, c1)
        got = dst.interior()[z0:z1].cpu().numpy()
        assert np.array_equal(got.view(np.uint64), want[1:-1, 1:-1, 1:-1].view(np.uint64)), (z0, z1)
    del src, dst
    torch.cuda.empty_cache()

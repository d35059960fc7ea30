"""The driver's direct stages, batched on the GPU.

The reference's ``evaluate`` runs three direct stages (driver.py:253 List 1,
:270 List 3close, :295 List 4close) through one closure,
``direct_stage(stage_name, list_csr)`` (driver.py:197-228): per target box,
gather the owned sources of the listed boxes (``_gather_sources``,
driver.py:109-113), add ``p2p`` for the box's conventional targets and one
``ts_accum`` per owned QBX center (target-specific mode).  Here the whole
stage is two launches:

* the box lists are expanded on the device into per-row source index lists
  (``tsqbx_box_rows_count/fill``, csrc/boxes.cu): one row per QBX center and
  one row per target box for the conventional targets;
* the centers go through the TSQBX evaluator (a ``TsqbxProblem``: the hot
  path, SELL layout, fast kernels), the conventional targets through the p2p
  row kernel (``P2PProblem.evaluate(rows=...)``).

Everything is in the tree's point order, exactly as the driver holds it
(``tree.points[SOURCES]``, permuted weights and normals, ``qcenters`` /
``qtargets``); the tree and list objects are duck-typed on the reference's
``Octree`` (``points``, ``owned_start``/``owned_end`` of shape (B, 3)) and
``_Csr`` (``starts``, ``flat``).  Like ``driver._ts_accum`` (driver.py:383-389)
nothing is validated.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as dv
from . import _lib
from .kernels import KernelSpec
from .nearlist import NearLists
from .p2p import P2PProblem
from .tsqbx import TsConfig, TsqbxProblem

SOURCES, TARGETS, CENTERS = 0, 1, 2      # tree.py:26-28


def _owner_rows(owned_start, owned_end, cls, n_points, is_target_box):
    """Boxes owning points of class ``cls`` in point order: (row_start (n_rows+1),
    row_box (n_rows,)); boxes outside the target-box set get row_box = -1."""
    s = np.asarray(owned_start[:, cls], dtype=np.int64)
    e = np.asarray(owned_end[:, cls], dtype=np.int64)
    boxes = np.nonzero(e > s)[0]
    boxes = boxes[np.argsort(s[boxes], kind="stable")]
    starts = s[boxes]
    ends = e[boxes]
    if n_points and (starts[0] != 0 or ends[-1] != n_points or np.any(starts[1:] != ends[:-1])):
        raise ValueError("owned point ranges do not partition the points")
    row_start = np.concatenate([starts, [n_points]]) if boxes.size else np.zeros(1, np.int64)
    row_box = np.where(is_target_box[boxes], boxes, -1).astype(np.int64)
    return row_start.astype(np.int64), row_box


@dv.on_device
def box_rows(row_box, list_starts, list_flat, box_src_start, box_src_end, device=None):
    """Device CSR (row_ptr int64, row_idx int32) of the concatenated owned source
    ranges of each row's box list (``tsqbx_box_rows_count/fill``)."""
    dev = dv.require_cuda(device)
    L = _lib.load()
    rb = dv.to_device(row_box, torch.int64, dev, (-1,))
    lp = dv.to_device(list_starts, torch.int64, dev, (-1,))
    lb = dv.to_device(list_flat, torch.int64, dev, (-1,))
    bs = dv.to_device(box_src_start, torch.int64, dev, (-1,))
    be = dv.to_device(box_src_end, torch.int64, dev, (-1,))
    n_rows = int(rb.shape[0])
    st = dv.stream_handle(dev)
    wsb = int(L.tsqbx_box_rows_workspace_bytes(n_rows))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    ptr = torch.empty(n_rows + 1, dtype=torch.int64, device=dev)
    total = torch.zeros(1, dtype=torch.int64, device=dev)
    _lib.check(L.tsqbx_box_rows_count(n_rows, rb.data_ptr(), lp.data_ptr(), dv.ptr(lb),
                                      bs.data_ptr(), be.data_ptr(), 1, ws.data_ptr(), wsb,
                                      ptr.data_ptr(), total.data_ptr(), st),
               "tsqbx_box_rows_count")
    n = int(total.item())
    idx = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    _lib.check(L.tsqbx_box_rows_fill(n_rows, rb.data_ptr(), lp.data_ptr(), dv.ptr(lb),
                                     bs.data_ptr(), be.data_ptr(), 1, ptr.data_ptr(),
                                     idx.data_ptr(), st), "tsqbx_box_rows_fill")
    return ptr, idx[:n]


class DirectStage:
    """One tree's direct stages on the GPU; ``run(list_csr)`` replaces one
    ``direct_stage(stage_name, list_csr)`` call of driver.py:197-228.

    ``weights`` are the permuted source weights ``w`` (driver.py:159),
    ``source_normals`` the permuted normals (D only), ``qtargets`` /
    ``qnormals`` the targets (and S' normals) of the tree-ordered centers,
    ``conv_normals`` the conventional targets' normals (S' only).

    The expansion of a list into row index lists, its SELL copy and the
    prepared TSQBX / p2p problems are built on the first ``run`` of that list
    and kept: the driver re-evaluates the same tree for every GMRES matvec
    (``prepared``, driver.py:118-122), so later calls only repack the sources
    when ``set_weights`` gave a new density and launch the two kernels.
    """

    @dv.on_device
    def __init__(self, spec: KernelSpec, p_qbx: int, tree, target_boxes, weights,
                 source_normals=None, qtargets=None, qnormals=None, conv_normals=None,
                 device=None):
        self.dev = dv.require_cuda(device)
        spec = self.spec = KernelSpec.coerce(spec)
        self.cfg = TsConfig(spec, int(p_qbx))
        dev = self.dev
        self.sources = dv.to_device(tree.points[SOURCES], torch.float64, dev, (-1, 3))
        self.weights = dv.to_device(weights, torch.complex128, dev, (-1,))
        self.snormals = (None if source_normals is None else
                         dv.to_device(source_normals, torch.float64, dev, (-1, 3)))
        self.conv = dv.to_device(tree.points[TARGETS], torch.float64, dev, (-1, 3))
        self.conv_normals = (None if conv_normals is None else
                             dv.to_device(conv_normals, torch.float64, dev, (-1, 3)))
        self.qcenters = dv.to_device(tree.points[CENTERS], torch.float64, dev, (-1, 3))
        self.qtargets = (self.qcenters if qtargets is None else
                         dv.to_device(qtargets, torch.float64, dev, (-1, 3)))
        self.qnormals = (None if qnormals is None else
                         dv.to_device(qnormals, torch.float64, dev, (-1, 3)))
        owned_start = np.asarray(tree.owned_start)
        owned_end = np.asarray(tree.owned_end)
        n_boxes = owned_start.shape[0]
        is_tb = np.zeros(n_boxes, dtype=bool)
        is_tb[np.asarray(target_boxes, dtype=np.int64)] = True
        self.box_src_start = np.ascontiguousarray(owned_start[:, SOURCES])
        self.box_src_end = np.ascontiguousarray(owned_end[:, SOURCES])
        n_c = int(self.qcenters.shape[0])
        n_t = int(self.conv.shape[0])
        c_start, c_box = _owner_rows(owned_start, owned_end, CENTERS, n_c, is_tb)
        self.center_box = np.repeat(c_box, np.diff(c_start))          # row box per center
        self.row_tgt, self.tbox = _owner_rows(owned_start, owned_end, TARGETS, n_t, is_tb)
        self.p2p = (P2PProblem(spec, self.sources, self.weights, self.snormals, dev)
                    if n_t else None)
        self._plans = {}
        self._version = 0

    @dv.on_own_device
    def set_weights(self, weights) -> None:
        """A new (permuted) density for the same tree: sources are repacked lazily."""
        self.weights = dv.to_device(weights, torch.complex128, self.dev, (-1,))
        if self.p2p is not None:
            self.p2p.set_weights(self.weights)
        self._version += 1

    def _plan(self, list_csr):
        key = id(list_csr)
        plan = self._plans.get(key)
        if plan is not None and plan["list"] is list_csr:
            return plan
        starts, flat = (list_csr.starts, list_csr.flat) if hasattr(list_csr, "starts") \
            else list_csr
        dev = self.dev
        n_c = int(self.qcenters.shape[0])
        plan = {"list": list_csr, "prob": None, "rows": None, "nts": 0, "version": self._version}
        if n_c:
            ptr, idx = box_rows(self.center_box, starts, flat, self.box_src_start,
                                self.box_src_end, dev)
            plan["nts"] = int(idx.shape[0])
            if plan["nts"]:
                near = NearLists(n_ctr=n_c, n_src=int(self.sources.shape[0]),
                                 n_pairs=plan["nts"], ptr=ptr, csr_idx=idx)
                plan["prob"] = TsqbxProblem(self.cfg, self.sources, self.weights, self.qcenters,
                                            self.qtargets, near, source_normals=self.snormals,
                                            target_normals=self.qnormals, device=dev)
        if self.p2p is not None and self.tbox.size:
            rptr, ridx = box_rows(self.tbox, starts, flat, self.box_src_start,
                                  self.box_src_end, dev)
            if int(ridx.shape[0]):
                plan["rows"] = self.p2p.rows(self.row_tgt, rptr, ridx, int(self.conv.shape[0]))
        self._plans[key] = plan
        return plan

    @dv.on_own_device
    def run(self, list_csr):
        """(conv_near, qbx_near_val, ts_pairs): the stage's additions to the
        driver's accumulators (complex128 CUDA tensors over the tree-ordered
        conventional targets and centers) and the ``counts["ts"]`` increment."""
        plan = self._plan(list_csr)
        dev = self.dev
        if plan["prob"] is not None:
            if plan["version"] != self._version:
                plan["prob"].set_weights(self.weights)
                plan["version"] = self._version
            qbx_add = plan["prob"].evaluate(validate=False).clone()
        else:
            qbx_add = torch.zeros(int(self.qcenters.shape[0]), dtype=torch.complex128,
                                  device=dev)
        if plan["rows"] is not None:
            # the reference's p2p raises on a coincident pair even inside the
            # driver (_core.pyx:109-111), so this one is screened
            conv_add = self.p2p.evaluate(self.conv, self.conv_normals, rows=plan["rows"],
                                         validate=True)
        else:
            conv_add = torch.zeros(int(self.conv.shape[0]), dtype=torch.complex128, device=dev)
        return conv_add, qbx_add, plan["nts"]

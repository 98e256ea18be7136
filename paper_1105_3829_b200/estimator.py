"""scikit-learn front end (the reference's estimator.py:13-108).

`MedianFilter2D(window, rank, percentile, max_error, mode, profile,
count_ops, bands)`: `fit` fixes the tree topology (uniform modes need only
the bit depth; "adaptive" learns value-frequency splits from the fitted
image), `transform` filters on the GPU and returns an array of the input's
shape and dtype.  Same parameters, validation order and errors as the
reference; `counters_` holds the (zero-tally) OpCounters of the last call.
"""

from __future__ import annotations

import numpy as np
from sklearn.base import BaseEstimator, TransformerMixin
from sklearn.utils.validation import check_is_fitted

from .engine import filter_image
from .topology import resolve_topology
from .validation import as_gray_image, check_max_error, check_window, resolve_rank


class MedianFilter2D(BaseEstimator, TransformerMixin):
    def __init__(self, window: int = 3, rank=None, percentile=None, max_error: int = 1,
                 mode: str = "uniform", profile=None, count_ops: bool = False, bands: int = 1):
        self.window = window
        self.rank = rank
        self.percentile = percentile
        self.max_error = max_error
        self.mode = mode
        self.profile = profile
        self.count_ops = count_ops
        self.bands = bands

    def _checked(self, X):
        img = as_gray_image(np.asarray(X))
        n = check_window(self.window, img.width, img.height)
        resolve_rank(n, self.rank, self.percentile)
        check_max_error(self.max_error)
        return img, n

    def fit(self, X, y=None):
        img, n = self._checked(X)
        self.bit_depth_ = img.bit_depth
        self.topology_ = resolve_topology(img, n, self.mode, self.profile)
        return self

    def transform(self, X):
        check_is_fitted(self, "topology_")
        img, n = self._checked(X)
        if img.bit_depth != self.bit_depth_:
            raise ValueError(f"transform input is {img.bit_depth}-bit, fitted on {self.bit_depth_}-bit")
        out, self.counters_ = filter_image(
            img, n, rank=self.rank, percentile=self.percentile, max_error=self.max_error,
            mode=self.mode, topology=self.topology_, counting=self.count_ops, bands=self.bands)
        return out.pixels

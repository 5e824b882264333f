"""B200-native (sm_100a) segmentation core for arXiv 1903.12294.

Drop-in for the data-parallel hot path of the reference package `mfseg`:
`engine.run` and its steps (windowed assignment, accumulation, centre update,
convergence) plus feature materialisation (merge, relabel, voxel bucketing,
statistics).  The compute lives in libmfseg_sm100.so (C ABI:
include/mfseg_sm100.h); this package is the host-side mirror of the
reference's Python interface.
"""

from .model import (ClusterCenter, ClusterParams, DomainExtent, FieldSet, ParameterError,
                    PointSet, Segmentation, interval_distances, space_time_distance)
from .engine import (CenterGrid, CenterState, accumulate, assign_iteration, field_distance,
                     has_converged, initial_assignment, max_center_delta, point_distance, run,
                     seed_centers, update_centers)
from .ingest import (IngestError, LinkIndex, NormalizationRecord, build_link_index,
                     domain_extent, load_field_device, normalize_variables, write_field)
from .postproc import (Feature, FeatureStats, build_features, feature_stats, merge_clusters,
                       merge_eligible)
from .pipeline import segment, segment_from_files
from . import artifacts

__all__ = [
    "CenterGrid", "CenterState", "ClusterCenter", "ClusterParams", "DomainExtent", "Feature",
    "FeatureStats", "FieldSet", "IngestError", "LinkIndex", "NormalizationRecord",
    "ParameterError", "PointSet", "Segmentation", "accumulate", "assign_iteration",
    "build_features", "build_link_index", "domain_extent", "feature_stats", "field_distance",
    "has_converged", "initial_assignment", "interval_distances", "max_center_delta",
    "merge_clusters", "merge_eligible", "normalize_variables", "point_distance", "run",
    "seed_centers", "segment", "space_time_distance", "update_centers", "artifacts",
    "load_field_device", "write_field", "segment_from_files",
]

__version__ = "0.1.0"
